"""Rank source lines of an `ncu --page source --csv --print-source cuda,sass` dump by
stall samples or warp instructions, with each line's share of the lost lane slots
(32 x instructions - thread instructions).  Usage: ncu_source_lines.py dump.csv samples|inst [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
cur = None; out = []
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0] in ("Function Name", "Line No"): continue
    if r[0] != "" and len(r) > 9:
        try:
            samp = float(r[4]) if r[4] not in ("-", "") else 0; inst = float(r[7]) if r[7] not in ("-","") else 0; tinst = float(r[8]) if r[8] not in ("-","") else 0
        except ValueError: continue
        if inst: out.append((cur, int(r[0]), r[1][:90], samp, inst, tinst))
tot_s = sum(o[3] for o in out); tot_i = sum(o[4] for o in out); tot_lost = sum(32*o[4]-o[5] for o in out)
print(f"total samples {tot_s:.4g} warp-inst {tot_i:.4g} lost lane slots {tot_lost:.4g} lane eff {1-tot_lost/(32*tot_i):.3f}")
key = {"samples":3, "inst":4}[sys.argv[2]] if len(sys.argv) > 2 else 3
for o in sorted(out, key=lambda o: -o[key])[:int(sys.argv[3]) if len(sys.argv) > 3 else 40]:
    lost = 32*o[4]-o[5]
    print(f"{o[3]/tot_s*100:5.1f}% samp {o[4]/tot_i*100:5.1f}% inst {lost/tot_lost*100:5.1f}% lost  {o[0]}:{o[1]}  {o[2]}")
