"""Per-source-line hot spots of an ncu report (run here): warp-stall samples and warp instructions per CUDA
line, from `ncu -i REP --page source --csv --print-source cuda,sass`.  Usage: ncu_lines.py REP [TOP]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
lines = []
fname = ""
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0] not in ("", "Line No") and r[0].isdigit():
        try:
            lines.append((int(r[4]), int(r[7]), fname, int(r[0]), r[1].strip()[:90]))
        except ValueError:
            pass
tot_s = sum(l[0] for l in lines) or 1
tot_i = sum(l[1] for l in lines) or 1
print(f"total samples {tot_s}  warp instructions {tot_i}")
for s, i, f, n, src in sorted(lines, reverse=True)[:top]:
    print(f"{100*s/tot_s:5.1f}% smp {100*i/tot_i:5.1f}% ins  {f}:{n:<5d} {src}")
