cd /root/repo
timeout -s KILL 1200 python -m pytest tests/ -m gpu -q -x -p no:cacheprovider -k "not c4_slices and not c3_slices" > gpurun_out/r2c_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2c_tests.log
SWEEP_TAG=sweep_r2c bash scripts/knob_sweep.sh "reordered c4 16" "batched c4 4" "given c4 2" -- "TNB_X=0" "TNB_EPI_SPIN=1"
