# fused-staging check: GPU tests, then bench with fusion off / on
TNB_DEBUG_FUSE=1 timeout -s KILL 300 python -c "
import paper_2103_03074_b200 as tnb
from paper_2103_03074_b200 import engine
w = tnb.load_workload('c4'); engine.head_program(w.tn, w.tree, w.sliced, 'single')" 2>&1 | grep TNB_FUSE
timeout -s KILL 900 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider > gpurun_out/fuse_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/fuse_tests.log
for f in 0 1; do
  TNB_FUSE=$f timeout -s KILL 400 python bench.py --no-cpu --no-e2e --reuse 0 2>gpurun_out/fuse_bench_$f.err | tee gpurun_out/fuse_bench_$f.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['breakdown_step_ms']; print('fuse=$f value %.3f gemm_ms %.1f total %.1f (breakdown step: convert %.1f simt %.1f) clocks %s launches %s'%(d['value'], d['device_ms_per_step']['gemm'], d['device_ms_per_step']['total'], b['convert_ms'], b['simt_ms'], d['clocks']['sm_mhz'], d['gpu_launches']))"
  tail -2 gpurun_out/fuse_bench_$f.err
done
TNB_FUSE=1 timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_requests_srcunit_tex_op_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm --csv --log-file gpurun_out/fuseprof_1.csv python bench.py --steps 1 --warmup 0 --slices 1 --no-e2e --no-cpu --reuse 0 > gpurun_out/fuseprof_1.log 2>&1; echo "ncu rc=$?"
