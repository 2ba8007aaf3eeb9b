cd /root/repo
timeout -s KILL 900 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2f_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2f_tests.log
SWEEP_TAG=sweep_r2f TNB_DIAG_REPS=3 bash scripts/knob_sweep.sh "reordered c4 16" "batched c4 4" "given c4 2" -- "TNB_X=0"
