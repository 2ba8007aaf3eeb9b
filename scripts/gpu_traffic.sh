# DRAM bytes of every tcgen05 GEMM launch of one C4 bench slice (+tail)
timeout -s KILL 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_f16x3 --csv --log-file gpurun_out/gemm_traffic.csv python bench.py --steps 1 --warmup 0 --slices 1 --no-e2e --no-cpu --reuse 0 > gpurun_out/gemm_traffic.log 2>&1; echo "rc=$?"
