"""Sum an ncu launch list (gpu__time_duration.sum --csv) between marker kernels.
Usage: python tools/launch_phases.py launches.csv  -> per graph: create / preprocess / run kernel time"""
import csv
import sys

SC = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
rows = list(csv.reader(open(sys.argv[1])))
hdr, seq = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    seq.append((d["Kernel Name"].split("(")[0], float(d["Metric Value"].replace(",", "")) * SC[d["Metric Unit"]]))
phase, acc, out = None, {}, []
for k, ms in seq:
    if "k_pack" in k or "k_check_ids" in k:
        if acc:
            out.append(acc)
        acc = {}
        phase = "create"
    elif "k_hash_empty" in k or ("k_rowhash" in k and phase == "create"):
        phase = "preprocess"
    elif "k_init" in k:
        phase = "run"
    acc[phase] = acc.get(phase, 0.0) + ms
if acc:
    out.append(acc)
for i, a in enumerate(out):
    print(i, {k: round(v, 3) for k, v in a.items()})
