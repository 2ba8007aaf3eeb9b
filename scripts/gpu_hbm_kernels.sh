# DRAM bytes / duration / throughput of every non-GEMM kernel of one C4 slice
# (gather, permute, slice sum, staging, SIMT, analytics) -> achieved HBM GB/s
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:'^(?!.*gemm_f16x3)' --csv --log-file gpurun_out/hbm_kernels.csv python bench.py --steps 1 --warmup 0 --slices 1 --no-e2e --no-cpu --reuse 0 > gpurun_out/hbm_kernels.log 2>&1; echo "rc=$?"
