cd /root/repo
TNB_SCALE_GUARD_BITS=-1 TNB_DIAG_SKIP_WARM=1 timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:gemm_f16x3 -s 10 -c 1 -f -o gpurun_out/r2d_step401 python scripts/diag_tree.py reordered c4 16 > gpurun_out/r2d_step401.log 2>&1; echo "ncu 401 rc=$?"
SWEEP_TAG=sweep_r2d TNB_DIAG_REPS=4 bash scripts/knob_sweep.sh "given c4 2" -- "TNB_X=0" "TNB_MMA_ORDER=1" "TNB_X=0" "TNB_MMA_ORDER=1"
