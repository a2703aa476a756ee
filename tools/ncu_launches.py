"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel name."""
import csv
import json
import sys
from collections import defaultdict

path = sys.argv[1]
ONLY_OURS = "--all" not in sys.argv
rows = [r for r in csv.reader(open(path)) if r]
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Name" in r)
h = rows[hdr_i]
agg = defaultdict(lambda: defaultdict(float))
count = defaultdict(set)
for r in rows[hdr_i + 1:]:
    d = dict(zip(h, r))
    import re
    m = re.findall(r"([A-Za-z_]\w*)(?:<[^()]*>)?\(", d["Kernel Name"])
    name = m[0] if m else d["Kernel Name"][:40]
    if ONLY_OURS and not ("dg::" in d["Kernel Name"][:40] or "unnamed>::" in d["Kernel Name"][:30]):
        continue
    try:
        v = float(d["Metric Value"].replace(",", ""))
    except ValueError:
        continue
    agg[name][d["Metric Name"]] += v
    count[name].add(d["ID"])
tot = sum(a.get("gpu__time_duration.sum", 0) for a in agg.values())
out = {}
print(f"{'kernel':40s} {'launches':>8s} {'time_us':>10s} {'share':>7s} {'dram_MB/launch':>15s}")
for name, a in sorted(agg.items(), key=lambda x: -x[1].get("gpu__time_duration.sum", 0)):
    n = len(count[name])
    t = a.get("gpu__time_duration.sum", 0)
    dram = a.get("dram__bytes_read.sum", 0) + a.get("dram__bytes_write.sum", 0)
    out[name] = {"launches": n, "time_ns": t, "share": t / tot if tot else 0, "dram_bytes_per_launch": dram / n if n else 0}
    print(f"{name:40s} {n:8d} {t / 1e3:10.1f} {t / tot * 100 if tot else 0:6.1f}% {dram / n / 1e6 if n else 0:15.2f}")
if len(sys.argv) > 2 and sys.argv[2].endswith(".json"):
    json.dump(out, open(sys.argv[2], "w"), indent=1)
