set -x
nproc; lscpu | grep "Model name"; free -g | head -2
timeout -s KILL 900 python bench.py > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench rc=$?"; cat gpurun_out/bench1.json; tail -5 gpurun_out/bench1.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 1 --warmup 1 --slices 1 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_f16x3 -s 3 -c 1 -o gpurun_out/gemm_r1 python bench.py --steps 1 --warmup 1 --slices 1 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"; tail -3 gpurun_out/ncu_full.log
