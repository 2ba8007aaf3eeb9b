"""profiles/<round>/gemm_traffic.json from a per-launch GEMM capture of the
given C4 tree (scripts/gpu_evidence_r2.sh: diag_tree.py given c4 2 under
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,...):
    python scripts/make_traffic_json.py gpurun_out/ev2_gemm_given.csv profiles/r2/gemm_traffic.json \
        [gpurun_out/ev2_gemm_given.log]
With the TNB_DEBUG_GEMM log the algorithmic bytes (complex64 A + B + C of each
step: 8 (MK + KN + MN)) are recorded beside the DRAM bytes."""
import json
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
import gemm_roofline as G  # noqa: E402

ln = G.launches(sys.argv[1])
per = [{"ms": l["gpu__time_duration.sum"] * 1e3,
        "dram_bytes": l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0),
        "tensor_busy_pct": l.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")}
       for l in ln]
if len(sys.argv) > 3:
    st = G.steps(sys.argv[3])
    order = [x for x in st if x["hoisted"]]
    rest = [x for x in st if not x["hoisted"]]
    order += rest * max(1, (len(per) - len(order)) // max(1, len(rest)))
    for p, x in zip(per, order):
        m, n, k = x["M"], x["Np"] // 2, x["Kp"] // 2
        p.update(step=x["step"], M=m, N=n, K=k, algorithmic_bytes=8.0 * (m * k + k * n + m * n))
tot = sum(p["dram_bytes"] for p in per)
out = {"source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
                 "sm__pipe_tensor_cycles_active (scripts/gpu_evidence_r2.sh): every gemm_f16x3 launch of "
                 "scripts/diag_tree.py given c4 2 (two C4 head slices, the bench's per-step work; "
                 "scale-guard re-runs off so launches map 1:1 to steps)",
       "launches": len(per), "dram_bytes_total": tot, "dram_bytes_per_launch": tot / len(per),
       "ncu_ms_total": sum(p["ms"] for p in per), "per_launch": per}
if all("algorithmic_bytes" in p for p in per):
    alg = sum(p["algorithmic_bytes"] for p in per)
    out["algorithmic_bytes_per_launch"] = alg / len(per)
    out["dram_over_algorithmic"] = tot / alg
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(f"{len(per)} launches, {tot / 1e9:.1f} GB, {tot / len(per) / 1e9:.2f} GB/launch")
