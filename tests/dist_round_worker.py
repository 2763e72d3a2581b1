"""Worker of the multi-rank CPU test (tests/test_dist_cpu.py), started by bench.spawn_ranks -- the launcher
`bench.py --gpus N` uses -- as one process per rank under torch.distributed.run.  Each rank runs bench.run_round
on its shard with the oracle context double over gloo and rank 0 writes the merged best-k and the all-reduced
counts to argv[1] (.npz)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import bench  # noqa: E402
from test_dist_cpu import Args, OracleCtx, N_PER_RANK  # noqa: E402
from workloads import make_config  # noqa: E402


def main():
    out = sys.argv[1]
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    dist.init_process_group("gloo")
    torch.set_num_threads(1)
    spec = make_config(1, n=N_PER_RANK)
    ctx = OracleCtx(spec, N_PER_RANK, rank * N_PER_RANK, N_PER_RANK * world)
    merged = bench.run_round(ctx, 123, Args, dist, world)
    counts, _ = ctx.check()
    dist.all_reduce(counts)
    if rank == 0:
        np.savez(out, merged=merged.numpy(), counts=counts.numpy(), world=world)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
