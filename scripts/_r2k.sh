cd /root/repo
T=ev3; O=gpurun_out
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $O/${T}_launches_c4.csv python bench.py --steps 1 --warmup 1 --slices 1 --no-e2e --no-cpu --reuse 0 --batch-s1 0 --opt-plan 0 --reordered 0 --batch-slices 0 --double 0 > $O/${T}_launches_c4.log 2>&1; echo "launch list rc=$?"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
for spec in "given c4 2" "reordered c4 16" "batched c4 4"; do
  set -- $spec
  TNB_SCALE_GUARD_BITS=-1 TNB_DEBUG_GEMM=1 TNB_DIAG_SKIP_WARM=1 timeout -s KILL 900 ncu --metrics $M --clock-control none -k regex:gemm_f16x3 --csv --log-file $O/${T}_gemm_$1.csv python scripts/diag_tree.py $1 $2 $3 > $O/${T}_gemm_$1.log 2>&1; echo "gemm $1 rc=$?"
done
TNB_SCALE_GUARD_BITS=-1 TNB_DIAG_SKIP_WARM=1 timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:gemm_f16x3 -s 11 -c 1 -f -o $O/${T}_gemm_top python scripts/diag_tree.py given c4 1 > $O/${T}_ncu_full.log 2>&1; echo "ncu full rc=$?"
