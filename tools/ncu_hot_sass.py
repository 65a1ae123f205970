"""Top SASS instructions by warp-stall samples of the first kernel in an ncu report (with their
neighbourhood), to see where a kernel waits.  Usage: python tools/ncu_hot_sass.py REP [N]"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
si = hdr.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[2:] if len(r) == len(hdr)]
tot = sum(int(r[si]) for r in data)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 15
print("kernel:", rows[0][1], "samples:", tot)
for idx, r in sorted(enumerate(data), key=lambda x: -int(x[1][si]))[:n]:
    print(f"{100 * int(r[si]) / tot:5.1f}%  {idx:5d}  {r[1].strip()}")
