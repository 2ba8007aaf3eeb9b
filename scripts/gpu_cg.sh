timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k cgemm > gpurun_out/cg_cgemm.log 2>&1; echo "cgemm rc=$?"; tail -5 gpurun_out/cg_cgemm.log
for cg in 1 2; do TNB_CTA_GROUP=$cg timeout -s KILL 300 python scripts/gemm_l2_probe.py 15 12 14 2>&1 | tail -1; done
for cg in 1 2; do TNB_CTA_GROUP=$cg timeout -s KILL 300 python scripts/gemm_l2_probe.py 14 13 14 2>&1 | tail -1; done
TNB_CTA_GROUP=2 timeout -s KILL 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -k regex:gemm -c 1 python scripts/gemm_l2_probe.py 15 12 14 2>&1 | grep -E "dram__bytes|duration|tensor"
bash scripts/gpu_round.sh r5
