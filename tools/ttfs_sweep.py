#!/usr/bin/env python
"""Time-to-first-satisfying over seeds for spec overrides (GPU).  Reading experiments.
    python tools/ttfs_sweep.py CONFIG N SEEDS "override1;override2" ...   e.g. "lam_goal=0.025" "lr_pos=0.002"
Each override set is a comma-separated list of spec fields; checks every 10 steps, budget 1000 steps."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_11833_b200 import TampContext  # noqa: E402
from workloads import make_config  # noqa: E402

cfg, n, seeds = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
torch.cuda.set_device(0)
for ov in sys.argv[4:] or [""]:
    res = []
    for seed in range(seeds):
        spec = make_config(cfg, n=n)
        spec.ik_iters, spec.ik_seeds = 20, 8
        for kv in ov.split(","):
            if kv:
                k, v = kv.split("=")
                setattr(spec, k, type(getattr(spec, k))(v))
        ctx = TampContext(spec, n)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.sample(seed=1000 * cfg + seed)
        hit, sat = None, 0
        for s in range(10, 1001, 10):
            c, _ = ctx.optimize_check(10)
            k = int(c[-2].item())
            if k > 0 and hit is None:
                hit = (s, time.perf_counter() - t0)
            sat = k
        res.append((hit, sat))
    ok = [h for h, _ in res if h]
    print(f"cfg {cfg} n {n} [{ov or 'defaults'}]: reached {len(ok)}/{seeds}; steps {[h[0] if h else None for h, _ in res]}; "
          f"s {[round(h[1], 3) if h else None for h, _ in res]}; satisfying at 1000: {[s for _, s in res]}", flush=True)
