"""Top SASS instructions by warp-stall samples for one kernel of an .ncu-rep.
Usage: python tools/ncu_hot.py <rep> <kernel-regex> [top=25]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ia, isrc, ist = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[2:] if len(r) == len(hdr) and r[ist].isdigit()]
tot = sum(int(r[ist] or 0) for r in body) or 1
for r in sorted(body, key=lambda r: -int(r[ist] or 0))[:top]:
    print(f"{int(r[ist]) / tot * 100:5.1f}%  {r[ia][-5:]}  {r[isrc].strip()[:90]}")
