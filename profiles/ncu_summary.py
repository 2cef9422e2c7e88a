"""Summarise an ncu --set full report of the ring kernel (run here, no GPU needed).
usage: python profiles/ncu_summary.py gpurun_out/<tag>_ring.ncu-rep [tokens_per_launch]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__cluster_dim_x", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__cycles_elapsed.avg.per_second",
        "local_load", "lts__t_bytes.sum"]
out = {}
for w in want:
    for i, h in enumerate(hdr):
        if h == w:
            out[w] = (vals[i], units[i])
for k, (v, u) in out.items():
    print(f"{k:60s} {v} {u}")
print("-- stall reasons (warps per issue) --")
st = []
for i, h in enumerate(hdr):
    if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
        try:
            st.append((float(vals[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        except ValueError:
            pass
for v, n in sorted(st, reverse=True)[:10]:
    print(f"  {n:30s} {v:.3f}")
if len(sys.argv) > 2:
    T = float(sys.argv[2])
    rd = float(out["dram__bytes_read.sum"][0]) * (1e9 if out["dram__bytes_read.sum"][1] == "Gbyte" else 1e6 if out["dram__bytes_read.sum"][1] == "Mbyte" else 1)
    wr = float(out["dram__bytes_write.sum"][0]) * (1e9 if out["dram__bytes_write.sum"][1] == "Gbyte" else 1e6 if out["dram__bytes_write.sum"][1] == "Mbyte" else 1)
    print(f"dram bytes per token: {(rd + wr) / T:.0f}")
