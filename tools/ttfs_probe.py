#!/usr/bin/env python
"""Where the time-to-first-satisfying goes (GPU): wall time of sample and of each optimize_check + host read, for
one config / N, three repetitions.  Usage: python tools/ttfs_probe.py CONFIG N"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_11833_b200 import TampContext  # noqa: E402
from workloads import make_config  # noqa: E402

cfg, n = int(sys.argv[1]), int(sys.argv[2])
torch.cuda.set_device(0)
spec = make_config(cfg, n=n)
spec.ik_iters, spec.ik_seeds = 20, 8
ctx = TampContext(spec, n)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.sample(seed=1000 * cfg + rep)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    marks = []
    for s in range(10, 101, 10):
        c, _ = ctx.optimize_check(10)
        k = int(c[-2].item())
        marks.append((s, round((time.perf_counter() - t1) * 1e3, 3), k))
        if k:
            break
    print(f"rep {rep}: sample+IK {1e3 * (t1 - t0):.3f} ms; (steps, ms since sample, satisfying): {marks}", flush=True)
