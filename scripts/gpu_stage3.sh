for cfg in "11 5" "10 5" "11 6" "10 4" "11 4"; do
  set -- $cfg
  echo "tile=$1 run=$2"
  TNB_STAGE_TILE=$1 TNB_STAGE_RUN=$2 timeout -s KILL 300 python bench.py --no-cpu --no-e2e --reuse 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(' value %.3f convert %.1f gemm %.1f clocks %s'%(d['value'], d['device_ms_per_step']['convert_ms'], d['device_ms_per_step']['gemm'], d['clocks']['sm_mhz']))"
done
