# tests + bench + launch list + one full ncu capture of the largest GEMM; $1 = tag
TAG=${1:-r}
bash scripts/gpu_round.sh $TAG
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_f16x3 -s 11 -c 1 -o gpurun_out/gemm_$TAG python bench.py --steps 1 --warmup 1 --slices 1 --no-e2e --no-cpu > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"; tail -2 gpurun_out/ncu_full_$TAG.log
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 8 -c 1 -o gpurun_out/stage_$TAG python bench.py --steps 1 --warmup 1 --slices 1 --no-e2e --no-cpu > gpurun_out/ncu_stage_$TAG.log 2>&1; echo "ncu stage rc=$?"
