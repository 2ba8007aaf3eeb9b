# Round evidence (one gpurun call): GPU tests, smoke, default bench, ncu launch
# list, per-GEMM DRAM traffic, one full ncu capture of the top GEMM launch.
T=${1:-ev}
timeout -s KILL 900 python -m pytest tests/ -m gpu -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${T}_tests.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${T}_smoke.log
timeout -s KILL 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"; cut -c1-400 gpurun_out/${T}_bench.json
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 1 --warmup 1 --slices 1 --no-e2e --no-cpu --reuse 0 --batch-s1 0 --opt-plan 0 --reordered 0 --batch-slices 0 > gpurun_out/${T}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout -s KILL 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_requests_srcunit_tex_op_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_f16x3 --csv --log-file gpurun_out/${T}_traffic.csv python bench.py --steps 1 --warmup 0 --slices 1 --no-e2e --no-cpu --reuse 0 --batch-s1 0 --opt-plan 0 --reordered 0 --batch-slices 0 > gpurun_out/${T}_traffic.log 2>&1; echo "ncu traffic rc=$?"
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:gemm_f16x3 -s 11 -c 1 -f -o gpurun_out/${T}_gemm_top python bench.py --steps 1 --warmup 0 --slices 1 --no-e2e --no-cpu --reuse 0 --batch-s1 0 --opt-plan 0 --reordered 0 --batch-slices 0 > gpurun_out/${T}_ncu_full.log 2>&1; echo "ncu full rc=$?"
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,power.limit --format=csv > gpurun_out/${T}_gpu.txt
