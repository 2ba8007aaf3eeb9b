"""Key metrics of an ncu --set full report (one or more kernels)."""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__sass_inst_executed_op_shared_st.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "smsp__average_warp_latency_issue_stalled",
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for vals in rows[2:]:
        name = vals[h.index("Kernel Name")][:90]
        print(f"== {name}")
        for i, k in enumerate(h):
            if any(k == w or k.startswith(w) for w in KEYS) or ("pipe_tensor" in k and "pct" in k and "realtime" not in k) \
                    or (k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")):
                try:
                    if float(vals[i].replace(",", "")) == 0:
                        continue
                except ValueError:
                    pass
                print(f"  {k} [{units[i]}] = {vals[i]}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
