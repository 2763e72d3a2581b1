"""Small end-to-end run of every libtamp kernel for compute-sanitizer (memcheck / racecheck / synccheck)."""
import sys
sys.path.insert(0, ".")
import torch
from workloads import make_config
from paper_2411_11833_b200 import TampContext

torch.cuda.set_device(0)
for cfg, lanes, selfc in [(1, 8, False), (2, 16, True), (4, 4, False), (3, 8, False), (1, 1, False), (6, 8, False)]:
    spec = make_config(cfg, n=40)
    spec.ik_iters = 3
    spec.self_collision = selfc
    ctx = TampContext(spec, 40, lanes_per_particle=lanes)
    ctx.sample(seed=1)
    ctx.optimize(2)
    counts, _ = ctx.check(cls=torch.empty(40, dtype=torch.uint8, device="cuda"))
    rec = ctx.best_k(4)
    ctx.merge_best_k(torch.cat([rec, rec]), 4)
    ctx.eval()
    torch.cuda.synchronize()
print("sanitize run ok")
