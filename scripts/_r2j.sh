cd /root/repo
timeout -s KILL 1500 python -m pytest tests/ -m gpu -q -rs -p no:cacheprovider > gpurun_out/r2j_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/r2j_tests.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2j_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2j_smoke.log
