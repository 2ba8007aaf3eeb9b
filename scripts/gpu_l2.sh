for cfg in "256 16" "128 16" "64 16" "0 16" "256 1000000" "256 4" "256 32"; do
  set -- $cfg
  TNB_L2_PROMO=$1 TNB_GROUP_M=$2 timeout -s KILL 300 python scripts/gemm_l2_probe.py 15 12 14 2>&1 | tail -1
  TNB_L2_PROMO=$1 TNB_GROUP_M=$2 timeout -s KILL 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -k regex:gemm -c 1 python scripts/gemm_l2_probe.py 15 12 14 2>&1 | grep -E "dram__bytes|duration|tensor" 
done
