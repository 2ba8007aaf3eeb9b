for cfg in "16 8" "8 8" "4 8" "8 16" "8 4"; do
  set -- $cfg
  echo "group_m=$1 chunk=$2"
  TNB_GROUP_M=$1 TNB_CHUNK_KB=$2 timeout -s KILL 300 python bench.py --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(' value %.3f gemm %.1f tensor_frac %.3f clocks %s'%(d['value'], d['roofline']['achieved'], d['roofline']['tensor_frac'], d['clocks']))"
done
TNB_GROUP_M=8 timeout -s KILL 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second -k regex:gemm -s 11 -c 1 python bench.py --steps 1 --warmup 1 --slices 1 --no-e2e --no-cpu 2>&1 | grep -E "dram__bytes|duration|tensor|per_second"
TNB_GROUP_M=16 timeout -s KILL 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second -k regex:gemm -s 11 -c 1 python bench.py --steps 1 --warmup 1 --slices 1 --no-e2e --no-cpu 2>&1 | grep -E "dram__bytes|duration|tensor|per_second"
