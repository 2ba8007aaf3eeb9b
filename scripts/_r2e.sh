cd /root/repo
timeout -s KILL 1200 python -m pytest tests/ -m gpu -q -x -p no:cacheprovider -k "not c4_slices and not c3_slices" > gpurun_out/r2e_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2e_tests.log
SWEEP_TAG=sweep_r2e TNB_DIAG_REPS=3 bash scripts/knob_sweep.sh "reordered c4 16" "batched c4 4" "given c4 2" -- "TNB_X=0"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
for spec in "reordered c4 16" "batched c4 4"; do
  set -- $spec
  TNB_SCALE_GUARD_BITS=-1 TNB_DEBUG_GEMM=1 TNB_DIAG_SKIP_WARM=1 timeout -s KILL 900 ncu --metrics $M --clock-control none -k regex:gemm_f16x3 --csv --log-file gpurun_out/r2e_gemm_$1.csv python scripts/diag_tree.py $1 $2 $3 > gpurun_out/r2e_gemm_$1.log 2>&1; echo "gemm $1 rc=$?"
  python scripts/gemm_roofline.py gpurun_out/r2e_gemm_$1.log gpurun_out/r2e_gemm_$1.csv > gpurun_out/r2e_gemm_$1_roofline.txt 2>&1; tail -4 gpurun_out/r2e_gemm_$1_roofline.txt
done
