"""Satisfied count of every hard term along an optimisation run (which constraints keep a skeleton from being
satisfied).  GPU.  Usage: python tools/term_trace.py CONFIG [N] [STEPS] [IK_ITERS] [SEED]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2411_11833_b200 import TampContext  # noqa: E402
from workloads import make_config  # noqa: E402

cfg = int(sys.argv[1])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
ik = int(sys.argv[4]) if len(sys.argv) > 4 else 20
seed = int(sys.argv[5]) if len(sys.argv) > 5 else 1
torch.cuda.set_device(0)
spec = make_config(cfg, n=n)
spec.ik_iters = ik
for kv in os.environ.get("SPEC_OVERRIDES", "").split(","):   # e.g. SPEC_OVERRIDES=lr_conf=0.003,lr_pos=0.002
    if kv:
        k, v = kv.split("=")
        setattr(spec, k, type(getattr(spec, k))(v))
ctx = TampContext(spec, n)
ctx.sample(seed=seed)
names = [f"{k}@{a}" for k, a in zip(ctx.term_kinds, ctx.term_actions)]
rows = []
for s in range(0, steps + 1, 100):
    if s:
        ctx.optimize(100)
    counts, _ = ctx.check()
    c = counts.cpu().numpy()
    rows.append(c)
    print(f"step {s:5d}  satisfying {c[-2]:7d}  invalid {c[-1]:5d}  min-term {names[int(np.argmin(c[:-2]))]} {c[:-2].min()}")
print("per term at the end (satisfied of", n, "):")
for nm, v0, v1 in zip(names, rows[0][:-2], rows[-1][:-2]):
    print(f"  {nm:14s} {v0:7d} -> {v1:7d}")
# particles that miss exactly one term: which term, and by how much (Jc / eps)
J, soft, Jc, _ = ctx.eval()
Jc = Jc.cpu().numpy()[:, :ctx.n_hard]
eps = np.array([spec.eps[k] for k in ctx.term_kinds])
miss = Jc > eps[None, :]
one = miss.sum(axis=1) == 1
print("particles missing exactly one term:", int(one.sum()), " two:", int((miss.sum(axis=1) == 2).sum()))
if one.any():
    which = np.argmax(miss[one], axis=1)
    for t in np.unique(which):
        sel = Jc[one][which == t, t]
        print(f"  {names[t]:14s} {int((which == t).sum()):6d} particles, J_c median {np.median(sel):.4g} (eps {eps[t]:.3g})")
# distribution of each Kin position residual among the particles that miss it
for t, nm in enumerate(names):
    if nm.startswith("KP"):
        bad = Jc[:, t] > eps[t]
        if bad.any():
            q = np.quantile(Jc[bad, t], [0.1, 0.5, 0.9])
            print(f"  {nm:8s} missed by {int(bad.sum()):6d}: J_c quantiles 10/50/90 % = {q[0]:.4f} {q[1]:.4f} {q[2]:.4f} m")
