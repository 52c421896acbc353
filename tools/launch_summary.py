"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file):
python tools/launch_summary.py launches.csv"""
import csv
import sys
from collections import defaultdict

tot, cnt = defaultdict(float), defaultdict(int)
for r in csv.reader(open(sys.argv[1])):
    if len(r) > 14 and r[12] == "gpu__time_duration.sum":
        v = float(r[14]) * (1e-3 if r[13] == "ns" else 1.0 if r[13] == "usecond" else 1e3 if r[13] == "msecond" else 1.0)
        tot[r[4]] += v
        cnt[r[4]] += 1
T = sum(tot.values()) or 1.0
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{tot[k] / T * 100:6.2f}%  {cnt[k]:4d} launches  {tot[k] / cnt[k] / 1e3:9.3f} ms avg  {k[:90]}")
