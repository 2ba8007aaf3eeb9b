# tensor-core threshold sweep (TNB_TC_MIN_RANK) at C5_26 (S=8) and C4 (S=2)
for wl in c5_26 c4; do
  S=2; [ "$wl" = "c5_26" ] && S=8
  for r in 27 25 23 21; do
    TNB_TC_MIN_RANK=$r timeout -s KILL 300 python bench.py --workload $wl --slices $S --no-cpu --no-e2e --reuse 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); b=d['breakdown_step_ms']
print('$wl min_rank $r value %.2f gemm %.1f non_gemm %.1f simt %.1f convert %.1f launches %d' % (d['value'], d['device_ms_per_step']['gemm'], d['device_ms_per_step']['non_gemm'], b['simt_ms'], b['convert_ms'], d['gpu_launches']))"
  done
done
