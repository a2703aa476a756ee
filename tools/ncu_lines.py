"""Per-CUDA-source-line instruction / stall totals of one kernel launch in an ncu report.
usage: python tools/ncu_lines.py REP [launch_index] [ntop]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
li = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda", "--launch-skip", str(li),
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
print(rows[0][:2])
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] in ("#", "Line", "Address"))
h = rows[hdr_i]
data = [dict(zip(h, r)) for r in rows[hdr_i + 1:] if len(r) == len(h)]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


ic = "Instructions Executed"
st = "Warp Stall Sampling (All Samples)"
ti = sum(f(d.get(ic, 0)) for d in data) or 1
ts = sum(f(d.get(st, 0)) for d in data) or 1
print(f"total warp-instr {ti:.0f}  samples {ts:.0f}")
for d in sorted(data, key=lambda d: -f(d.get(ic, 0)))[:ntop]:
    print(f"inst {f(d[ic]) / ti * 100:5.1f}%  stall {f(d[st]) / ts * 100:5.1f}%  L{d.get('#', d.get('Line', '?')):>5s} {d['Source'].strip()[:100]}")
