"""Instructions / stall samples of an ncu report per source-line range of a file (code regions named by the first line
of each range).  Usage: ncu_regions.py REP FILE START:NAME [START:NAME ...]   (lines >= START until the next START;
code inlined from other files is attributed to the last region seen in address order)"""
import csv
import subprocess
import sys

rep, fname = sys.argv[1], sys.argv[2]
marks = sorted((int(a.split(":")[0]), a.split(":", 1)[1]) for a in sys.argv[3:])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
f, cur, sass = "", None, []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0].isdigit():
        cur = (f, int(r[0]))
        continue
    if len(r) > 8 and r[0] == "" and r[2].startswith("0x"):
        try:
            sass.append((int(r[2], 16), cur, int(r[7]), int(r[4])))
        except ValueError:
            pass
sass.sort()
tot, region = {}, "other"
for addr, line, ins, smp in sass:
    if line and line[0] == fname:
        region = "before"
        for st, nm in marks:
            if line[1] >= st:
                region = nm
    t = tot.setdefault(region, [0, 0])
    t[0] += ins
    t[1] += smp
ti = sum(v[0] for v in tot.values()) or 1
ts = sum(v[1] for v in tot.values()) or 1
for k, v in sorted(tot.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:24s} {100 * v[0] / ti:6.1f}% inst {100 * v[1] / ts:6.1f}% samples")
