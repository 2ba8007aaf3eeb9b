# bench twice (no CPU baseline / e2e / reuse) and print the key numbers
for i in 1 2; do timeout -s KILL 400 python bench.py --no-cpu --no-e2e --reuse 0 2>gpurun_out/bq_$i.err > gpurun_out/bq_$i.json; python -c "
import json; d=json.load(open('gpurun_out/bq_$i.json')); m=d['device_ms_per_step']; b=d.get('breakdown_step_ms', {})
print('value %.3f total %.1f gemm %.1f non_gemm %.1f clocks %s | breakdown step: %s' % (d['value'], m['total'], m['gemm'], m.get('non_gemm', 0), d['clocks']['sm_mhz'], {k: round(v, 1) for k, v in b.items() if k != 'note'}))"; done
