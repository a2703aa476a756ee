"""Basic-block instruction / stall breakdown of one kernel in an ncu report (SASS source page).
usage: python tools/ncu_blocks.py REP [ntop]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h) and r[0] != "Address"]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


# the page may repeat the kernel; keep the first copy (addresses restart)
seen = set()
k = []
for d in data:
    if d["Address"] in seen:
        break
    seen.add(d["Address"])
    k.append(d)
ic, st = "Instructions Executed", "Warp Stall Sampling (All Samples)"
ti = sum(f(d[ic]) for d in k) or 1
ts = sum(f(d[st]) for d in k) or 1
print(f"kernel: {len(k)} SASS, {ti:.0f} warp-instr, {ts:.0f} stall samples")
blocks, cur = [], None
for i, d in enumerate(k):
    c = f(d[ic])
    if cur and c == cur["cnt"] and c > 0:
        cur["end"] = i
        cur["n"] += 1
        cur["stall"] += f(d[st])
    else:
        if cur:
            blocks.append(cur)
        cur = {"start": i, "end": i, "cnt": c, "n": 1, "stall": f(d[st]), "first": d["Source"].strip()}
blocks.append(cur)
for b in sorted(blocks, key=lambda b: -(b["cnt"] * b["n"]))[:ntop]:
    print(f"[{b['start']:5d}-{b['end']:5d}] n={b['n']:4d} x{b['cnt']:9.0f} = {b['cnt'] * b['n'] / ti * 100:5.1f}% inst"
          f"  {b['stall'] / ts * 100:5.1f}% stall  {b['first'][:60]}")
