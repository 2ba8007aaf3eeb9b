for wl in c5_26 c4; do
  S=2; [ "$wl" = "c5_26" ] && S=8
  TNB_DEBUG_FUSE=1 timeout -s KILL 300 python -c "
import paper_2103_03074_b200 as tnb
from paper_2103_03074_b200 import engine
w = tnb.load_workload('$wl'); p = engine.head_program(w.tn, w.tree, w.sliced, 'single'); print('$wl fused', p.info.n_steps_fused, 'fast', p.info.n_steps_fused_fast)" 2>&1 | grep -E "smallk|fused"
  timeout -s KILL 300 python bench.py --workload $wl --slices $S --no-cpu --no-e2e --reuse 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); b=d['breakdown_step_ms']
print('$wl value %.2f gemm %.1f non_gemm %.1f simt %.1f convert %.1f launches %d' % (d['value'], d['device_ms_per_step']['gemm'], d['device_ms_per_step']['non_gemm'], b['simt_ms'], b['convert_ms'], d['gpu_launches']))"
done
timeout -s KILL 900 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
