"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel: launches,
total and mean duration, share of the total.

    python tools/summarize_launches.py launches.csv [out.csv]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0].replace("qsr::<unnamed>::", "")
    v = float(d["Metric Value"].replace(",", ""))
    if d.get("Metric Unit") == "msecond":
        v *= 1e6
    elif d.get("Metric Unit") == "usecond":
        v *= 1e3
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(t for _, t in agg.values())
lines = ["kernel,launches,total_ms,mean_us,share"]
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    lines.append(f"{k},{c},{t / 1e6:.3f},{t / c / 1e3:.2f},{t / tot:.4f}")
out = "\n".join(lines)
print(out)
if len(sys.argv) > 2:
    open(sys.argv[2], "w").write(out + "\n")
