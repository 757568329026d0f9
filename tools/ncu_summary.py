"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per-kernel totals."""
import csv
import sys
from collections import defaultdict

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"')))
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
tot, cnt = defaultdict(float), defaultdict(int)
seen = 0
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    seen += 1
    if seen <= skip:
        continue
    name = r["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").replace("fetigpu::", "")
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    v = v / 1000.0 if unit in ("nsecond", "ns") else (v if unit in ("usecond", "us") else v * 1000.0)
    tot[name] += v
    cnt[name] += 1
grand = sum(tot.values())
print(f"{'kernel':40s} {'launches':>8s} {'total us':>10s} {'avg us':>9s} {'share':>6s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:40s} {cnt[k]:8d} {tot[k]:10.1f} {tot[k]/cnt[k]:9.2f} {tot[k]/grand:6.1%}")
print(f"{'TOTAL':40s} {sum(cnt.values()):8d} {grand:10.1f}")
