cd /root/repo
timeout -s KILL 900 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py tests/test_gpu_treeopt.py tests/test_gpu_slice_batch.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2g_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2g_tests.log
TNB_DEBUG_FUSE=1 TNB_DIAG_SKIP_WARM=1 timeout 300 python scripts/diag_tree.py reordered c4 1 2>&1 | grep -E "TNB_FUSE step (401|403|395) " | head
SWEEP_TAG=sweep_r2g TNB_DIAG_REPS=3 bash scripts/knob_sweep.sh "reordered c4 16" "batched c4 4" -- "TNB_X=0"
