for pace in 0 256 0 512 64; do
  echo "pace=$pace"
  TNB_PACE=$pace timeout -s KILL 300 python bench.py --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(' value %.3f gemm %.1f tensor_frac %.3f clocks %s'%(d['value'], d['roofline']['achieved'], d['roofline']['tensor_frac'], d['clocks']))"
done
