# iteration check: GPU parity tests, skinny-shape probe, two bench runs
set -u
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/iter_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/iter_tests.log
timeout -s KILL 600 python scripts/gemm_probe.py shapes ${PROBE_SHAPES:-11,19,7 8,22,8 13,17,8 10,6,20 7,14,16 13,17,10 15,12,15} 2>&1 | tee gpurun_out/iter_probe.log
for i in 1 2; do timeout -s KILL 300 python bench.py --no-cpu --reuse 0 > gpurun_out/iter_bench$i.json 2>gpurun_out/iter_bench$i.err; python -c "import json,sys; d=json.loads(open('gpurun_out/iter_bench$i.json').read()); print(' value %.3f e2e %.3f gemm_ms %.1f convert %.1f simt %.1f clocks %s'%(d['value'], d['e2e']['value'], d['device_ms_per_step']['gemm'], d['device_ms_per_step']['convert_ms'], d['device_ms_per_step']['simt_ms'], d['clocks']['sm_mhz']))"; done
