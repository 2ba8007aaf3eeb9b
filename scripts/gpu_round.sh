# tests + bench + launch list (one gpurun call); $1 = tag
TAG=${1:-r}
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/tests_$TAG.log
timeout -s KILL 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; cat gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 1 --slices 1 --no-e2e --no-cpu > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu rc=$?"
