"""Stall samples / instructions of the TS kernel grouped by warp role (SASS regions located by
marker instructions).  usage: python tools/ncu_roles.py REP"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h) and r[0] != "Address"]
seen, k = set(), []
for d in data:
    if d["Address"] in seen:
        break
    seen.add(d["Address"])
    k.append(d)


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


stc = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
# region starts: first index of each marker
marks = {}
for i, d in enumerate(k):
    src = d["Source"]
    for name, pat in (("producer", "UBLKCP"), ("producer", "UTMALDG"), ("mma", "UTCIMMA"), ("unpack", "STTM"),
                      ("epilogue", "LDTM")):
        if pat in src:
            marks.setdefault(name, []).append(i)
print({n: (min(v), max(v)) for n, v in marks.items()})
# assign each instruction to the nearest marker region (by position) - coarse
cuts = sorted((min(v), n) for n, v in marks.items())
tot_s = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in k)
tot_i = sum(f(d["Instructions Executed"]) for d in k)
bounds = [(0, "prologue")] + cuts
for j, (st, name) in enumerate(bounds):
    en = bounds[j + 1][0] if j + 1 < len(bounds) else len(k)
    seg = k[st:en]
    s = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in seg)
    ins = sum(f(d["Instructions Executed"]) for d in seg)
    agg = {}
    for d in seg:
        for c in stc:
            agg[c[6:]] = agg.get(c[6:], 0) + f(d[c])
    top = sorted(agg.items(), key=lambda x: -x[1])[:4]
    print(f"{name:10s} [{st:5d},{en:5d}) samples {s / tot_s * 100:5.1f}%  inst {ins / tot_i * 100:5.1f}%  " +
          ", ".join(f"{a}={b / max(s, 1) * 100:.0f}%" for a, b in top))
