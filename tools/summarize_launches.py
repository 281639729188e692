"""Summarise an ncu launch list (--metrics gpu__time_duration.sum[,dram__bytes_read.sum,
dram__bytes_write.sum] --csv) by kernel: launches, total and mean duration, share of the total,
and DRAM bytes per launch when captured.

    python tools/summarize_launches.py launches.csv [out.csv]
"""
import collections
import csv
import sys

UNIT = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
per_launch = collections.defaultdict(dict)  # (kernel, id) -> metric -> value
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    name = d["Kernel Name"].split("(")[0].replace("qsr::<unnamed>::", "").replace("<unnamed>::", "")
    v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d.get("Metric Unit", ""), 1.0)
    per_launch[(name, d.get("ID", ""))][d["Metric Name"]] = v
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for (name, _), m in per_launch.items():
    if "gpu__time_duration.sum" not in m:
        continue
    a = agg[name]
    a[0] += 1
    a[1] += m["gpu__time_duration.sum"]
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tot = sum(t for _, t, _ in agg.values())
lines = ["kernel,launches,total_ms,mean_us,share,dram_bytes_per_launch"]
for k, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    lines.append(f"{k},{c},{t / 1e6:.3f},{t / c / 1e3:.2f},{t / tot:.4f},{b / c:.4g}")
out = "\n".join(lines)
print(out)
if len(sys.argv) > 2:
    open(sys.argv[2], "w").write(out + "\n")
