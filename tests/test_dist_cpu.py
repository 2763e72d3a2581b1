"""Multi-rank host logic of bench.py on CPU: world size 2 over gloo (127.0.0.1).

Each rank runs `bench.run_round` on its shard with a context double whose arithmetic is the oracle
(test infrastructure); the test checks the collective wiring of SURVEY §8(e): the all-reduced counts
equal the single-process counts over all particles, and the all-gathered + merged best-k equals the
global best-k (global indices from the rank offsets)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import tamp_oracle as O
from workloads import make_config

N_PER_RANK, WORLD, K, STEPS = 24, 2, 5, 4


class OracleCtx:
    """Stand-in for TampContext with the same methods bench.run_round calls."""

    def __init__(self, spec, n, gofs, n_global):
        self.spec, self.n, self.gofs, self.n_global = spec, n, gofs, n_global
        self.csp = O.build_csp(spec)
        self.D = self.csp.D

    def sample(self, seed):
        x, g = O.initialize_particles(self.spec, self.csp, seed, np.arange(self.gofs, self.gofs + self.n))
        self.st = O.new_state(x, g)

    def optimize(self, k):
        O.optimize(self.spec, self.csp, self.st, k, 1.0 / self.n_global)

    def check(self, cls=None, counts=None):
        _, c, *_ = O.check(self.spec, self.csp, self.st)
        return torch.tensor(c, dtype=torch.int32), cls

    def optimize_check(self, k, cls=None, counts=None):      # tamp_optimize_and_check: optimize, then check
        self.optimize(k)
        return self.check(cls, counts)

    def best_k(self, k, out=None):
        cls, _, J, soft, _ = O.check(self.spec, self.csp, self.st)
        sel, kc, kcost = O.best_k(cls, J, soft, np.arange(self.gofs, self.gofs + self.n), k)
        return torch.tensor(records(kc, kcost, sel + self.gofs, self.st.x[sel]))

    def merge_best_k(self, rec, k):
        r = rec.numpy()
        gidx = r[:, 2].copy().view(np.uint32).astype(np.int64) | (r[:, 3].copy().view(np.int32).astype(np.int64) << 32)
        order = np.lexsort((gidx, r[:, 1], r[:, 0]))[:k]
        return torch.tensor(r[order])


def records(cls, cost, gidx, x):
    out = np.zeros((len(cls), x.shape[1] + 4), np.float32)
    out[:, 0] = cls
    out[:, 1] = cost
    out[:, 2] = (gidx & 0xFFFFFFFF).astype(np.uint32).view(np.float32)
    out[:, 3] = (gidx >> 32).astype(np.int32).view(np.float32)
    out[:, 4:] = x
    return out


class Args:
    adam_steps = STEPS
    check_every = 2
    k = K


def _worker(rank, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    import bench
    torch.set_num_threads(1)
    spec = make_config(1, n=N_PER_RANK)
    ctx = OracleCtx(spec, N_PER_RANK, rank * N_PER_RANK, N_PER_RANK * WORLD)
    merged = bench.run_round(ctx, 123, Args, dist, WORLD)
    counts, _ = ctx.check()
    dist.all_reduce(counts)
    if rank == 0:
        q.put((merged.numpy(), counts.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_round_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    merged, counts = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single process over all particles
    spec = make_config(1, n=N_PER_RANK * WORLD)
    one = OracleCtx(spec, N_PER_RANK * WORLD, 0, N_PER_RANK * WORLD)
    one.sample(123)
    one.optimize(STEPS)
    c1, _ = one.check()
    ref = one.best_k(K).numpy()
    np.testing.assert_array_equal(counts, c1.numpy())
    np.testing.assert_array_equal(merged[:, :4], ref[:, :4])
    np.testing.assert_allclose(merged[:, 4:], ref[:, 4:], rtol=0, atol=0)


def _single_process_reference():
    spec = make_config(1, n=N_PER_RANK * WORLD)
    one = OracleCtx(spec, N_PER_RANK * WORLD, 0, N_PER_RANK * WORLD)
    one.sample(123)
    one.optimize(STEPS)
    c1, _ = one.check()
    return c1.numpy(), one.best_k(K).numpy()


def test_bench_launcher_two_ranks(tmp_path):
    """The launcher of `bench.py --gpus N` (bench.spawn_ranks: torch.distributed.run, one process per rank,
    127.0.0.1) starting a world of 2 gloo ranks that run bench.run_round: same counts and best-k as one process."""
    import bench
    out = str(tmp_path / "r.npz")
    rc = bench.spawn_ranks(WORLD, [out], script=os.path.join(os.path.dirname(__file__), "dist_round_worker.py"))
    assert rc == 0
    r = np.load(out)
    assert int(r["world"]) == WORLD
    c1, ref = _single_process_reference()
    np.testing.assert_array_equal(r["counts"], c1)
    np.testing.assert_array_equal(r["merged"], ref)


def test_bench_gpus_2_reference_arm_through_the_launcher():
    """`python bench.py --gpus 2 --impl reference` without torchrun: bench spawns 2 ranks itself (gloo for the
    host-only reference arm); rank 0 prints the JSON line with n_gpus = 2, the other rank exits 0."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--impl", "reference",
                        "--config", "1", "--steps", "1", "--warmup", "0"], capture_output=True, text=True, env=env,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"


def test_bench_refuses_mismatched_world_size():
    """--gpus N under a launcher that started a different number of ranks fails loudly."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--impl", "reference"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr
