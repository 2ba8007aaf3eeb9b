# quick iteration: fused-edge plan, GPU tests, bench x2, per-GEMM ncu, launch list
TNB_DEBUG_FUSE=1 timeout -s KILL 300 python -c "
import paper_2103_03074_b200 as tnb
from paper_2103_03074_b200 import engine
w = tnb.load_workload('c4'); p = engine.head_program(w.tn, w.tree, w.sliced, 'single'); print('fused', p.info.n_steps_fused, 'fast', p.info.n_steps_fused_fast, 'kernels/slice', p.info.kernels_per_slice)" 2>&1 | grep -E "TNB_FUSE|fused" | sed 's/nvec.*lane_w/lane_w/'
timeout -s KILL 900 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider > gpurun_out/it_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/it_tests.log
bash scripts/gpu_bench_quick.sh
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/it_launches.csv python bench.py --steps 1 --warmup 1 --slices 1 --no-e2e --no-cpu --reuse 0 > /dev/null 2>&1; echo "ncu rc=$?"; python scripts/launch_summary.py gpurun_out/it_launches.csv | head -12
