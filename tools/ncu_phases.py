"""Attribute every SASS instruction of the profiled kernel to a phase of k_particle (by address order: an
inlined helper's code belongs to the kernel-body line that precedes it) and print instructions / stall
samples per phase.  Usage: ncu_phases.py REP"""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname, cur_line, sass = "", None, []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0].isdigit():
        cur_line = (fname, int(r[0]))
        continue
    if len(r) > 8 and r[0] == "" and r[2].startswith("0x"):
        try:
            sass.append((int(r[2], 16), cur_line, int(r[7]), int(r[4]), r[3].strip()))
        except ValueError:
            pass
sass.sort()
# phase boundaries: kernel-body line numbers of particle.cuh (first line of each phase)
src = open("paper_2411_11833_b200/csrc/particle.cuh").read().split("\n")
marks = []
for i, l in enumerate(src, 1):
    for key, name in (("// ---- phase A", "A instances"), ("// ---- phase B", "B FK loop"),
                      ("// robot spheres vs OBBs", "B coll OBB"), ("// robot spheres vs movable", "B coll objects"),
                      ("// robot self-collision", "B self"), ("Wrench Wl[LPL]", "B wrench"),
                      ("// held object at a MoveHold", "B held"), ("// Kin(q, o, g, p)", "B kin"),
                      ("// joint limits:", "B JL"), ("// suffix sums of link", "B backward"),
                      ("// ---- phase C", "C place"), ("// ---- phase D", "D soft"),
                      ("// ---- phase E", "E inst grads"), ("// ---- phase F", "F adam")):
        if key in l:
            marks.append((i, name))
k_start = min(i for i, l in enumerate(src, 1) if "k_particle(" in l and "__global__" in "".join(src[i - 3:i]))
marks.sort()


def phase_of(line):
    if line is None or line[0] != "particle.cuh" or line[1] < k_start:
        return None
    name = "setup"
    for i, n in marks:
        if line[1] >= i:
            name = n
    return name


tot = {}
cur = "setup"
for addr, line, ins, smp, op in sass:
    ph = phase_of(line)
    if ph is not None:
        cur = ph
    t = tot.setdefault(cur, [0, 0])
    t[0] += ins
    t[1] += smp
ti = sum(v[0] for v in tot.values()) or 1
ts = sum(v[1] for v in tot.values()) or 1
print(f"{'phase':16s} {'warp inst %':>12s} {'samples %':>10s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:16s} {100 * v[0] / ti:12.1f} {100 * v[1] / ts:10.1f}")

if len(sys.argv) > 2:      # top source lines of one phase
    want = sys.argv[2]
    agg = {}
    cur = "setup"
    for addr, line, ins, smp, op in sass:
        ph = phase_of(line)
        if ph is not None:
            cur = ph
        if cur == want:
            a = agg.setdefault(line, [0, 0])
            a[0] += ins
            a[1] += smp
    for line, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:25]:
        txt = src[line[1] - 1].strip()[:80] if line and line[0] == "particle.cuh" else ""
        print(f"{100 * v[0] / ti:6.2f}% ins {100 * v[1] / ts:6.2f}% smp {line} {txt}")

# static code size per phase (SASS instructions x 16 B)
stat = {}
cur = "setup"
for addr, line, ins, smp, op in sass:
    ph = phase_of(line)
    if ph is not None:
        cur = ph
    stat[cur] = stat.get(cur, 0) + 1
print("static code per phase (KB):", {k: round(v * 16 / 1024, 1) for k, v in sorted(stat.items(), key=lambda kv: -kv[1])})
