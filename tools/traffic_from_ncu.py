"""Record the DRAM traffic of one kernel from an `ncu --set full` report into
profiles/gather_traffic.json (read by bench.py for roofline.traffic).
Usage: python tools/traffic_from_ncu.py <rep> <kernel-regex> <key e.g. rmat-24:reduced> <source note>"""
import csv
import json
import os
import re
import subprocess
import sys

rep, kern, key, note = sys.argv[1:5]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
for vals in rows[2:]:
    d = dict(zip(hdr, vals))
    if not re.search(kern, d.get("Kernel Name", "")):
        continue
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = float(d["dram__bytes_read.sum"].replace(",", "")) * scale[units[hdr.index("dram__bytes_read.sum")]]
    wr = float(d["dram__bytes_write.sum"].replace(",", "")) * scale[units[hdr.index("dram__bytes_write.sum")]]
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "gather_traffic.json")
    pj = json.load(open(path)) if os.path.exists(path) else {}
    def num(k):
        try:
            return float(d[k].replace(",", ""))
        except (KeyError, ValueError):
            return None
    pj[key] = {"dram_bytes_per_launch": int(rd + wr), "dram_read_bytes": int(rd), "dram_write_bytes": int(wr),
               "l2_hit_rate_pct": num("lts__t_sector_hit_rate.pct"),
               "l1tex_to_l2_request_busy_pct": num("l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed"),
               "kernel": d["Kernel Name"][:80], "source": note}
    json.dump(pj, open(path, "w"), indent=1)
    print(key, pj[key])
    break
else:
    sys.exit(f"no kernel matching {kern}")
