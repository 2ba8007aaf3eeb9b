cd /root/repo
t0=$(date +%s); timeout -s KILL 1700 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2h_ref.json 2> gpurun_out/r2h_ref.err; echo "ref rc=$? wall $(( $(date +%s) - t0 )) s"; cut -c1-500 gpurun_out/r2h_ref.json
t0=$(date +%s); timeout -s KILL 1700 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err; echo "bench rc=$? wall $(( $(date +%s) - t0 )) s"; cut -c1-300 gpurun_out/r2h_bench.json
