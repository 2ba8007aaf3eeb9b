cd /root/repo
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
TNB_SCALE_GUARD_BITS=-1 TNB_DEBUG_GEMM=1 TNB_DIAG_SKIP_WARM=1 timeout -s KILL 900 ncu --metrics $M --clock-control none -k regex:gemm_f16x3 --csv --log-file gpurun_out/r2r_gemm_plan.csv python scripts/diag_tree.py plan c4_opt31_b200 1 > gpurun_out/r2r_gemm_plan.log 2>&1; echo "rc=$?"
TNB_SCALE_GUARD_BITS=-1 TNB_DIAG_SKIP_WARM=1 timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2r_all_plan.csv python scripts/diag_tree.py plan c4_opt31_b200 1 > /dev/null 2>&1; echo "rc=$?"
