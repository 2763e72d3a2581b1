"""Stick Button on the GPU (SURVEY f4 + f3): optimise the stick skeleton and the infeasible direct-press
skeleton, print the per-constraint satisfied counts (Eq. 5 inputs), then run Algorithm 1 over both."""
import sys
import time

import torch

from paper_2411_11833_b200 import TampContext, plan_heuristic
import paper_2411_11833_b200.planner as planner
from workloads import make_config

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
torch.cuda.set_device(0)
for cfg in (6, 7):
    spec = make_config(cfg, n=n)
    spec.ik_iters = 20
    ctx = TampContext(spec, n)
    ctx.sample(seed=1)
    c0, _ = ctx.check()
    print(cfg, "terms", ctx.term_kinds)
    print(cfg, "init counts", c0.tolist(), "H", plan_heuristic(c0.cpu(), ctx.n_hard, -1e6))
    for it in range(100):
        ctx.optimize(10)
        c, _ = ctx.check()
        if int(c[-2]) > 0 or it % 25 == 24:
            print(cfg, "step", 10 * (it + 1), c.tolist())
        if int(c[-2]) > 0:
            break
specs = [make_config(7, n=n), make_config(6, n=n)]
for s in specs:
    s.ik_iters = 20
t = time.time()
res = planner.cutamp(specs, n, seed=5, steps_per_pop=200, max_pops=10, k=4)
torch.cuda.synchronize()
print("planner", None if res is None else (res.skeleton, res.steps, res.pops, res.heuristics), time.time() - t)
