"""Small end-to-end run of every libtamp kernel variant (device-check builds: tools/device_checks.sh; compute-sanitizer
when available).  Usage: python tools/sanitize_small.py [path/to/libtamp.so]"""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
from workloads import make_config  # noqa: E402
from paper_2411_11833_b200 import TampContext, load  # noqa: E402

if len(sys.argv) > 1:
    load(sys.argv[1])
torch.cuda.set_device(0)
cases = [(1, 8, False, 0), (2, 16, True, 0), (4, 4, False, 0), (3, 8, False, 0), (1, 1, False, 0), (6, 8, False, 0),
         (4, 16, False, 0), (4, 16, True, 0), (4, 16, False, 640), (3, 8, False, 896), (3, 8, False, 1024),
         (3, 8, True, 0), (2, 8, False, 768),
         (7, 8, False, 0), (5, 8, False, 512), (1, 1, False, 640), (1, 1, False, 96), (2, 1, False, 0)]
for cfg, lanes, selfc, threads in cases:
    n = 300
    spec = make_config(cfg, n=n)
    spec.ik_iters, spec.ik_seeds = 3, 4
    spec.self_collision = selfc and lanes != 1
    ctx = TampContext(spec, n, lanes_per_particle=lanes, block_threads=threads)
    ctx.sample(seed=1)
    ctx.optimize(2)
    ctx.optimize_check(3, cls=torch.empty(n, dtype=torch.uint8, device="cuda"))
    counts, _ = ctx.check(cls=torch.empty(n, dtype=torch.uint8, device="cuda"))
    rec = ctx.best_k(4)
    ctx.merge_best_k(torch.cat([rec, rec]), 4)
    ctx.eval()
    torch.cuda.synchronize()
    print(f"config {cfg} lanes {ctx.lanes_per_particle} threads {ctx.block_threads} self {spec.self_collision}: ok",
          flush=True)
print("all cases ok")
