set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q -k "cgemm" -p no:cacheprovider > gpurun_out/gpu1_cgemm.log 2>&1; echo "cgemm rc=$?"
tail -30 gpurun_out/gpu1_cgemm.log
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -k "not cgemm" -p no:cacheprovider > gpurun_out/gpu1_rest.log 2>&1; echo "rest rc=$?"
tail -40 gpurun_out/gpu1_rest.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/gpu1_smoke.log 2>&1; echo "smoke rc=$?"; tail -5 gpurun_out/gpu1_smoke.log
