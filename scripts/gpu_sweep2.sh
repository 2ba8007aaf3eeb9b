for cfg in "16 64" "8 64" "32 64" "16 32" "8 32" "16 16"; do
  set -- $cfg
  echo "group_m=$1 pace=$2"
  TNB_GROUP_M=$1 TNB_PACE=$2 timeout -s KILL 300 python bench.py --no-cpu --no-e2e --reuse 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(' value %.3f gemm_ms %.1f gemm_tflops %.1f clocks %s'%(d['value'], d['device_ms_per_step']['gemm'], d['roofline']['achieved'], d['clocks']['sm_mhz']))"
done
