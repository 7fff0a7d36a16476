"""Per-source-line stall samples / instructions from an ncu report
(ncu --page source --csv --print-source cuda,sass).  Development aid."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
cur = None
out = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0] not in ("", "Line No"):
        try:
            out.append((float(r[4]), float(r[7]), cur, r[0], r[1][:100]))
        except ValueError:
            pass
tot = sum(o[0] for o in out) or 1
ti = sum(o[1] for o in out) or 1
out.sort(reverse=True)
for o in out[:top]:
    print(f"{o[0]/tot*100:5.1f}% samp {o[1]/ti*100:5.1f}% inst  {o[2]}:{o[3]}  {o[4]}")
