# quick iteration: fused-edge plan, GPU tests, bench, per-GEMM ncu times
TNB_DEBUG_FUSE=1 timeout -s KILL 300 python -c "
import paper_2103_03074_b200 as tnb
from paper_2103_03074_b200 import engine
w = tnb.load_workload('c4'); engine.head_program(w.tn, w.tree, w.sliced, 'single')" 2>&1 | grep TNB_FUSE | sed 's/nvec.*lane_w/lane_w/'
timeout -s KILL 900 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider > gpurun_out/it_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/it_tests.log
for i in 1 2; do timeout -s KILL 400 python bench.py --no-cpu --no-e2e --reuse 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value %.3f gemm_ms %.1f convert %.1f simt %.1f total %.1f clocks %s'%(d['value'], d['device_ms_per_step']['gemm'], d['device_ms_per_step']['convert_ms'], d['device_ms_per_step']['simt_ms'], d['device_ms_per_step']['total'], d['clocks']['sm_mhz']))"; done
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_requests_srcunit_tex_op_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_f16x3 --csv --log-file gpurun_out/it_traffic.csv python bench.py --steps 1 --warmup 0 --slices 1 --no-e2e --no-cpu --reuse 0 > gpurun_out/it_traffic.log 2>&1; echo "ncu rc=$?"
