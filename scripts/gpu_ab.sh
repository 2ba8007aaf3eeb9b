# A/B an env knob on the C4 bench: GPU tests once, then alternate A and B runs
# usage: KNOB=TNB_STAGE_ASYNC A=0 B=1 bash scripts/gpu_ab.sh
set -u
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ab_tests.log
for i in 1 2; do for v in $A $B; do
  env $KNOB=$v timeout -s KILL 300 python bench.py --no-cpu --reuse 0 --no-e2e > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/ab_$v.json').read()); m=d['device_ms_per_step']; print(' $KNOB=$v value %.3f gemm %.1f convert %.1f simt %.1f other %.1f clocks %s'%(d['value'], m['gemm'], m['convert_ms'], m['simt_ms'], m['other_ms'], d['clocks']['sm_mhz']))"
done; done
