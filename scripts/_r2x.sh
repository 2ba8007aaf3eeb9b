cd /root/repo
timeout -s KILL 1500 python -m pytest tests/ -m gpu -q -rs -p no:cacheprovider > gpurun_out/r2x_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2x_tests.log
bash scripts/bench_sweep.sh r2x
