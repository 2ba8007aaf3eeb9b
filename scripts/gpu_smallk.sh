timeout -s KILL 900 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider > gpurun_out/sk_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/sk_tests.log
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:smallk --csv --log-file gpurun_out/sk.csv python bench.py --steps 1 --warmup 0 --slices 1 --no-e2e --no-cpu --reuse 0 > /dev/null 2>&1; echo "ncu rc=$?"
bash scripts/gpu_bench_quick.sh
