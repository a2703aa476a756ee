"""Summarise an ncu report: key SOL metrics + top stalled SASS lines with stall reasons."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 20
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, vals = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed.sum", "sm__pipe_tensor_cycles_active", "sm__pipe_alu_cycles_active.avg.pct", "sm__inst_issued.avg.pct",
        "smsp__issue_active.avg.pct", "l1tex__data_pipe_lsu_wavefronts_mem_shared", "sm__cycles_elapsed.avg",
        "smsp__average_warp_latency_issue_stalled", "sm__pipe_fma_cycles_active.avg.pct", "gpu__dram_throughput.avg.pct",
        "sm__pipe_shared_cycles_active.avg.pct", "smsp__warps_active.avg"]
for i, name in enumerate(h):
    if any(w in name for w in want):
        print(f"{name:80s} {vals[i]:>20s} {units[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in data) or 1
stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
agg = {c: sum(f(d[c]) for d in data) for c in stall_cols}
print("stall reasons (% of samples):", ", ".join(f"{k[6:]}={v / tot * 100:.1f}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
for d in sorted(data, key=lambda d: -f(d["Warp Stall Sampling (All Samples)"]))[:ntop]:
    top = sorted(((f(d[c]), c[6:]) for c in stall_cols), reverse=True)[:2]
    print(f"{f(d['Warp Stall Sampling (All Samples)']) / tot * 100:5.1f}% x{d['Instructions Executed']:>9s} {d['Source'][:70]:70s} {top}")
