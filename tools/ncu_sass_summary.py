"""Summarise an `ncu --page source --csv --print-source sass` dump: instruction
mix, stall reasons and the hottest SASS regions (development aid)."""
import csv
import re
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]


def num(s):
    try:
        return float(s.replace(",", ""))
    except Exception:
        return 0.0


tot_inst = sum(num(d["Instructions Executed"]) for d in data)
tot_samp = sum(num(d["Warp Stall Sampling (All Samples)"]) for d in data)
print(f"total warp-instructions {tot_inst:.4g}, stall samples {tot_samp:.4g}")
mix = Counter()
for d in data:
    op = d["Source"].strip().split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1] if len(op) > 1 else o
    mix[o.split(".")[0]] += num(d["Instructions Executed"])
print("opcode mix (top 25):")
for o, c in mix.most_common(25):
    print(f"  {o:10s} {c/tot_inst*100:5.1f}%")
stalls = defaultdict(float)
for d in data:
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            stalls[k] += num(v)
print("stall reasons (% of samples):")
for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:10]:
    print(f"  {k:28s} {v/max(tot_samp,1)*100:5.1f}%")
# hottest 40-instruction windows by samples
W = 48
best = []
for i in range(0, len(data) - W, W // 2):
    s = sum(num(d["Warp Stall Sampling (All Samples)"]) for d in data[i:i + W])
    ins = sum(num(d["Instructions Executed"]) for d in data[i:i + W])
    best.append((s, ins, i))
best.sort(reverse=True)
print("hottest windows (samples%, inst%, start addr, first ops):")
for s, ins, i in best[:int(sys.argv[2]) if len(sys.argv) > 2 else 8]:
    ops = Counter(d["Source"].strip().split()[0].split(".")[0] for d in data[i:i + W] if d["Source"].strip())
    print(f"  {s/tot_samp*100:5.1f}% {ins/tot_inst*100:5.1f}% {data[i]['Address']} {dict(ops.most_common(6))}")
