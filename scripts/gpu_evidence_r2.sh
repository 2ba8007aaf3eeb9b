# Round-2 evidence (one gpurun call): tests, smoke, bench, headline launch list,
# per-GEMM roofline captures of the given / re-ordered / batched C4 trees, one
# full ncu capture of the top GEMM.  Outputs under gpurun_out/${T}_*.
T=${1:-ev2}
O=gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,power.limit --format=csv > $O/${T}_gpu.txt
if [ -z "$SKIP_TESTS" ]; then
timeout -s KILL 1200 python -m pytest tests/ -m gpu -q -rs -p no:cacheprovider > $O/${T}_tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/${T}_tests.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/${T}_smoke.log
fi
if [ -z "$SKIP_BENCH" ]; then
timeout -s KILL 1200 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench rc=$?"; cut -c1-300 $O/${T}_bench.json
fi
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $O/${T}_launches_c4.csv python bench.py --steps 1 --warmup 1 --slices 1 --no-e2e --no-cpu --reuse 0 --batch-s1 0 --opt-plan 0 --reordered 0 --batch-slices 0 > $O/${T}_launches_c4.log 2>&1; echo "launch list rc=$?"
for spec in "given c4 2" "reordered c4 16" "batched c4 4"; do
  set -- $spec
  TNB_SCALE_GUARD_BITS=-1 TNB_DEBUG_GEMM=1 TNB_DIAG_SKIP_WARM=1 timeout -s KILL 900 ncu --metrics $M --clock-control none -k regex:"gemm_(f16x3|skinny)" --csv --log-file $O/${T}_gemm_$1.csv python scripts/diag_tree.py $1 $2 $3 > $O/${T}_gemm_$1.log 2>&1; echo "gemm $1 rc=$?"
  python scripts/gemm_roofline.py $O/${T}_gemm_$1.log $O/${T}_gemm_$1.csv > $O/${T}_gemm_$1_roofline.txt 2>&1; tail -4 $O/${T}_gemm_$1_roofline.txt
done
if [ -z "$SKIP_FULL" ]; then
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:gemm_f16x3 -s 11 -c 1 -f -o $O/${T}_gemm_top python bench.py --steps 1 --warmup 0 --slices 1 --no-e2e --no-cpu --reuse 0 --batch-s1 0 --opt-plan 0 --reordered 0 --batch-slices 0 > $O/${T}_ncu_full.log 2>&1; echo "ncu full rc=$?"
fi
