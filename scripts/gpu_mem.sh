timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_io.py -q -x -p no:cacheprovider > gpurun_out/mem_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/mem_tests.log
python -c "
import paper_2103_03074_b200 as t
from paper_2103_03074_b200 import engine as E
for n in ['c4','c5_32']:
    w=t.load_workload(n); p=E.head_program(w.tn,w.tree,w.sliced,'single')
    i=p.info; print(n,'arena GiB %.1f persist GiB %.2f maxscratch GiB %.1f'%(i.arena_bytes/2**30,i.persistent_bytes/2**30,i.scratch_bytes/2**30)); del p; E.clear_cache()
"
timeout -s KILL 600 python bench.py --workload c5_32 --slices 1 --steps 3 --warmup 3 --no-cpu --no-e2e --reuse 1 2>&1 | tail -1 | cut -c1-400
timeout -s KILL 600 python bench.py --no-cpu --no-e2e --reuse 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(' value %.3f gemm_ms %.1f convert %.1f simt %.1f clocks %s'%(d['value'], d['device_ms_per_step']['gemm'], d['device_ms_per_step']['convert_ms'], d['device_ms_per_step']['simt_ms'], d['clocks']['sm_mhz']))"
