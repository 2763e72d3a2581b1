"""Time-to-first-satisfying of cuTAMP vs the paper's Optimization and Sampling baselines
on the synthetic workloads, through Algorithm 1 (planner.cutamp) on one GPU.  Wall-clock with a device sync;
prints one line per (config, method, trial)."""
import statistics
import sys
import time

import torch

import paper_2411_11833_b200.planner as planner
from workloads import make_config

cfgs = [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "1,2,6").split(",")]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
trials = int(sys.argv[3]) if len(sys.argv) > 3 else 3
torch.cuda.set_device(0)
# warm-up (context creation, module load)
planner.cutamp([make_config(1, n=256)], 256, steps_per_pop=10, max_pops=1)
for cfg in cfgs:
    for method in planner.METHODS:
        times, steps = [], []
        for trial in range(trials):
            spec = make_config(cfg, n=n)
            spec.ik_iters = 20
            spec.ik_seeds = 8
            torch.cuda.synchronize()
            t = time.perf_counter()
            res = planner.cutamp([spec], n, seed=1000 * cfg + trial, steps_per_pop=1000, max_pops=1, method=method)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
            times.append(dt if res is not None else float("inf"))
            steps.append(res.steps if res is not None else None)
        solved = [t for t in times if t != float("inf")]
        print(f"cfg {cfg} n {n} method {method:12s} solved {len(solved)}/{trials} "
              f"median_s {statistics.median(times) if solved else float('inf'):.4f} steps {steps}", flush=True)
