set -x
timeout -s KILL 300 python scripts/gemm_probe.py acc > gpurun_out/probe_acc.log 2>&1; echo "acc rc=$?"; cat gpurun_out/probe_acc.log
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider > gpurun_out/gpu2_tests.log 2>&1; echo "tests rc=$?"; tail -30 gpurun_out/gpu2_tests.log
timeout -s KILL 600 python scripts/gemm_probe.py perf > gpurun_out/probe_perf.log 2>&1; echo "perf rc=$?"; cat gpurun_out/probe_perf.log
