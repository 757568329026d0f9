"""Print key metrics per kernel from an ncu report: python tools/ncu_details.py rep.ncu-rep [regex]"""
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__waves_per_multiprocessor",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]
for d in data:
    name = d[hdr.index("Kernel Name")].split("(")[0]
    if pat and not pat.search(name):
        continue
    out = [name[-38:]]
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            out.append(f"{w.split('__')[1].split('.')[0][:22]}={d[i]}{units[i]}")
    print(" | ".join(out))
