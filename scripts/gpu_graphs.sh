# CUDA-graph segments: tests, then bench A/B (TNB_GRAPHS=0/1) at C4 and C5_26
timeout -s KILL 900 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
for g in 0 1; do
  for wl in c4 c5_26; do
    S=2; [ "$wl" = "c5_26" ] && S=8
    TNB_GRAPHS=$g timeout -s KILL 300 python bench.py --workload $wl --slices $S --no-cpu --no-e2e --reuse 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('graphs $g $wl value %.2f total %.1f gemm %.1f non_gemm %.1f launches %d' % (d['value'], d['device_ms_per_step']['total'], d['device_ms_per_step']['gemm'], d['device_ms_per_step']['non_gemm'], d['gpu_launches']))"
  done
done
