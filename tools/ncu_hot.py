"""Hottest SASS lines (warp-stall samples) of one kernel in an ncu report:
python tools/ncu_hot.py rep.ncu-rep kernel_regex [min_share] [launch_skip]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
share = float(sys.argv[3]) if len(sys.argv) > 3 else 0.01
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern, "-s", skip, "-c", "1",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, d = rows[1], rows[2:]
i, e = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
tot = sum(int(r[i]) for r in d if r[i].isdigit())
for n, r in enumerate(d):
    if r[i].isdigit() and int(r[i]) > tot * share:
        print(f"{n:5d} {int(r[i]) / tot:6.1%} {r[e]:>8s}  {r[1].strip()[:100]}")
print("total samples", tot, "instructions", len(d))
