# skinny / short-K GEMM shapes of the C4 head: timing + one ncu capture each
set -u
mkdir -p gpurun_out
timeout -s KILL 900 python scripts/gemm_probe.py shapes 11,19,7 8,22,8 13,17,8 10,6,20 7,14,16 13,17,10 > gpurun_out/skinny_probe.log 2>&1; echo "probe rc=$?"
cat gpurun_out/skinny_probe.log
for s in 11,19,7 10,6,20; do
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_f16x3 -s 1 -c 1 \
    -o gpurun_out/skinny_${s//,/_} python scripts/gemm_probe.py shapes $s > gpurun_out/ncu_skinny_${s//,/_}.log 2>&1; echo "ncu $s rc=$?"
done
