"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list per kernel.
Usage: python tools/launch_summary.py launches.csv [out.txt]"""
import collections
import csv
import sys

SCALE = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
cnt = collections.Counter()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    k = d["Kernel Name"].split("(")[0].replace("void ", "")[:70]
    v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1e-6)
    agg[k] = agg.get(k, 0.0) + v
    cnt[k] += 1
tot = sum(agg.values())
lines = [f"{'ms':>10} {'share':>6} {'launches':>8}  kernel", "-" * 90]
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    lines.append(f"{v:10.3f} {v / tot * 100:5.1f}% {cnt[k]:8d}  {k}")
lines.append(f"{tot:10.3f}  total over {sum(cnt.values())} launches (cold-cache, serialised by ncu)")
out = "\n".join(lines)
print(out)
if len(sys.argv) > 2:
    open(sys.argv[2], "w").write(out + "\n")
