# BASELINE configs[4]: m=20 slice-throughput sweep over the sliced-edge count
# (target space 2^26/2^28/2^30/2^32 -> n_e 63/58/53/48) and the batch size
# (2^20 vs 2^21 correlated bitstrings), XEB on the synthetic amplitudes.
# One JSON line per point in gpurun_out/sweep_<tag>.jsonl.
TAG=${1:-r}
OUT=gpurun_out/sweep_$TAG.jsonl
: > $OUT
for wl in c5_26 c5_28 c4 c5_32 c5_n21; do
  S=2
  [ "$wl" = "c5_26" ] && S=8
  [ "$wl" = "c5_28" ] && S=4
  [ "$wl" = "c5_32" ] && S=1
  timeout -s KILL 600 python bench.py --workload $wl --slices $S --steps 3 --warmup 3 --no-cpu --no-e2e --reuse 1 --double 0 >> $OUT 2> gpurun_out/sweep_${TAG}_$wl.err
  echo "$wl rc=$?"
done
python - <<EOF
import json
for line in open("$OUT"):
    d = json.loads(line)
    r = d.get("cross_slice_reuse") or {}
    o = d.get("reordered_same_slices") or {}
    print(f"{d['config']['workload'][:40]:40s} n_e? slices/s {d['value']:.3f} TFLOP/s {d['contraction_tflops']:.1f} "
          f"gemm {d['roofline']['achieved']:.0f} reuse {r.get('value', 0):.2f} xeb {d['xeb_partial_subset']:.4g} "
          f"reordered {o.get('slices_per_s', 0):.2f} ({o.get('executed_tflops', 0):.0f} TFLOP/s executed) "
          f"batched k={(d.get('batched_slices') or {}).get('batch_log2')} {(d.get('batched_slices') or {}).get('slices_per_s', 0):.1f} "
          f"({(d.get('batched_slices') or {}).get('executed_tflops', 0):.0f} TFLOP/s executed)")
EOF
