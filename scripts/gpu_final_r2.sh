# Round-2 final evidence on the final code: full GPU suite + smoke, driver-style
# bench (20 steps), per-launch GEMM roofline of the given / re-ordered / batched
# C4 trees.  Outputs gpurun_out/fin_*.
O=gpurun_out; T=fin
timeout -s KILL 1500 python -m pytest tests/ -m gpu -q -rs -p no:cacheprovider > $O/${T}_tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/${T}_tests.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/${T}_smoke.log
timeout -s KILL 1700 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench rc=$?"; cut -c1-300 $O/${T}_bench.json
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
for spec in "given c4 2" "reordered c4 16" "batched c4 4"; do
  set -- $spec
  TNB_SCALE_GUARD_BITS=-1 TNB_DEBUG_GEMM=1 TNB_DIAG_SKIP_WARM=1 timeout -s KILL 900 ncu --metrics $M --clock-control none -k regex:"gemm_(f16x3|skinny)" --csv --log-file $O/${T}_gemm_$1.csv python scripts/diag_tree.py $1 $2 $3 > $O/${T}_gemm_$1.log 2>&1; echo "gemm $1 rc=$?"
done
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $O/${T}_launches_c4.csv python bench.py --steps 1 --warmup 1 --slices 1 --no-e2e --no-cpu --reuse 0 --batch-s1 0 --opt-plan 0 --reordered 0 --batch-slices 0 --double 0 > $O/${T}_launches_c4.log 2>&1; echo "launch list rc=$?"
