"""Per-CUDA-source-line stall samples with the dominant reasons, sorted by samples (one kernel of an
ncu report, mixed cuda+sass source page).  usage: python tools/ncu_stall_lines.py REP [ntop]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
tot, fname, line, hdr = {}, "?", None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        cols = [i for i, c in enumerate(hdr) if c.startswith("stall_") and "Not Issued" not in c]
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    if r[0]:
        line = (fname, int(r[0]), r[1].strip()[:80])
        continue
    try:
        smp = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
        inst = float(r[hdr.index("Instructions Executed")])
    except ValueError:
        continue
    t = tot.setdefault(line, [0.0, 0.0, {}])
    t[0] += smp
    t[1] += inst
    for i in cols:
        try:
            v = float(r[i])
        except ValueError:
            continue
        if v:
            t[2][hdr[i][6:]] = t[2].get(hdr[i][6:], 0.0) + v
ts = sum(v[0] for v in tot.values()) or 1
print(f"samples {ts:.0f}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1][0])[:ntop]:
    rs = sorted(v[2].items(), key=lambda kv: -kv[1])[:3]
    print(f"{v[0] / ts * 100:5.1f}%  inst {v[1]:9.0f}  {k[0]}:{k[1]:<5d} {k[2][:60]:60s} " +
          " ".join(f"{n}={c / max(v[0], 1) * 100:.0f}%" for n, c in rs))
