"""Per-CUDA-source-line totals (instructions executed, stall samples) of one kernel in an ncu
report, from the mixed cuda+sass source page.  usage: python tools/ncu_srclines.py REP [ntop]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
tot = {}
fname = "?"
line = None
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:
        line = (fname, int(r[0]), r[1].strip()[:90])
        continue
    try:
        inst = float(r[7]); smp = float(r[4])
    except ValueError:
        continue
    t = tot.setdefault(line, [0.0, 0.0])
    t[0] += inst
    t[1] += smp
ti = sum(v[0] for v in tot.values()) or 1
ts = sum(v[1] for v in tot.values()) or 1
print(f"total warp-instr {ti:.0f}  samples {ts:.0f}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1][0])[:ntop]:
    print(f"inst {v[0] / ti * 100:5.1f}% ({v[0]:9.0f})  stall {v[1] / ts * 100:5.1f}%  {k[0]}:{k[1]:<5d} {k[2]}")
