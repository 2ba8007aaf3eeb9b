set -u
mkdir -p gpurun_out
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:stage_async -c 2 \
  -o gpurun_out/stage_async python scripts/gemm_probe.py shapes 15,12,15 > gpurun_out/ncu_stage_async.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_stage_async.log
