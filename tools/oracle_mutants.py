#!/usr/bin/env python
"""Mutation check of the oracle's pins: apply one-line mutants to a scratch copy of oracle/tamp_oracle.py and
run the CPU pin suites against each; every mutant must make at least one test fail.

    python tools/oracle_mutants.py [pytest files...]      (default: the oracle pin suites)
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITES = ["tests/test_oracle_pins.py", "tests/test_oracle_geometry.py", "tests/test_oracle_csp.py"]

# (name, original line fragment, mutated fragment)
MUTANTS = [
    ("SC shrink sign flipped", "lower = _t(s.lo)[None, :] + r[:, None]", "lower = _t(s.lo)[None, :] - r[:, None]"),
    ("SC upper shrink sign flipped", "upper = _t(s.hi)[None, :] - r[:, None]", "upper = _t(s.hi)[None, :] + r[:, None]"),
    ("TrajLength drops its endpoint confs",
     "seq = [conf((\"var\", q1))] + [conf((\"knot\", tv, j)) for j in range(V[tv].n_knots)] + [conf((\"var\", q2))]",
     "seq = [conf((\"knot\", tv, j)) for j in range(V[tv].n_knots)]"),
    ("lambda_goal dropped", "soft = soft + spec.lam_goal * obj_dist(P)", "soft = soft + obj_dist(P)"),
    ("held object attached by T(g) instead of T(g)^-1", "T_obj = frames[:, 8] @ inverse(G[:, gslot[gv]])",
     "T_obj = frames[:, 8] @ G[:, gslot[gv]]"),
    ("sphere -> link index shifted", "T = frames[:, torch.as_tensor(robot.sphere_link, dtype=torch.long)]",
     "T = frames[:, torch.as_tensor(robot.sphere_link, dtype=torch.long) - 1]"),
    ("CP without its support OBB exclusion", "obbs = [b for i, b in enumerate(spec.obbs) if i != s.support_obb]",
     "obbs = list(spec.obbs)"),
    ("CP without its support object exclusion", "Jc.append(scene_cost(w, r, t.scene, {t.obj, s.support_obj}, obbs))",
     "Jc.append(scene_cost(w, r, t.scene, {t.obj}, obbs))"),
]


def main():
    suites = sys.argv[1:] or SUITES
    src = open(os.path.join(ROOT, "oracle", "tamp_oracle.py")).read()
    ok = True
    for name, a, b in MUTANTS:
        assert src.count(a) == 1, f"mutant anchor not found exactly once: {name}"
        with tempfile.TemporaryDirectory() as tmp:
            for d in ("oracle", "tests", "workloads"):
                shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                                ignore=shutil.ignore_patterns("__pycache__"))
            shutil.copy(os.path.join(ROOT, "pytest.ini"), tmp)
            open(os.path.join(tmp, "oracle", "tamp_oracle.py"), "w").write(src.replace(a, b))
            r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "not gpu", "-p", "no:cacheprovider"]
                               + suites, cwd=tmp, capture_output=True, text=True)
            killed = r.returncode != 0
            failed = [ln.split(" ")[1] for ln in r.stdout.splitlines() if ln.startswith("FAILED")]
            print(f"{'KILLED ' if killed else 'SURVIVED'}  {name}  {failed[:1]}", flush=True)
            ok &= killed
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
