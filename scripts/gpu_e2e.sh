timeout -s KILL 600 python -m pytest tests/ -m gpu -q -x -p no:cacheprovider > gpurun_out/e2e_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/e2e_tests.log
timeout -s KILL 600 python scripts/e2e_profile.py 2>&1 | head -14
timeout -s KILL 300 python bench.py --no-cpu --reuse 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(' value %.3f e2e %.3f gemm_ms %.1f clocks %s'%(d['value'], d['e2e']['value'], d['device_ms_per_step']['gemm'], d['clocks']['sm_mhz']))"
