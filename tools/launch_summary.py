"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel launches, total and share of device time (development aid)."""
import csv
import re
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0] != "ID"]
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows:
    name = re.sub(r"\(.*", "", r[4]).replace("void ", "")
    tot[name] += float(r[-1])
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':70s} {'launches':>8s} {'total ms':>10s} {'share':>7s} {'avg ms':>9s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k[:70]:70s} {cnt[k]:8d} {v/1e6:10.2f} {v/T*100:6.1f}% {v/cnt[k]/1e6:9.3f}")
print(f"{'TOTAL':70s} {sum(cnt.values()):8d} {T/1e6:10.2f}")
