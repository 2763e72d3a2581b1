"""Algorithm 1 over candidate skeletons: the Eq. 5 heuristic orders the skeletons and the
loop returns satisfying particles of a feasible one.  CPU: the loop logic with the oracle standing in for
the GPU context; GPU: the real library."""
import copy

import numpy as np
import pytest
import torch

from oracle import tamp_oracle as O
from workloads import make_config
from workloads.scenes import Surface

import paper_2411_11833_b200.planner as planner


def _infeasible_variant(spec):
    """Same skeleton with the goal region moved 3 m away: StablePlace / Kin can never hold (zero counts)."""
    s = copy.deepcopy(spec)
    s.surfaces = [Surface("far", np.array([3.0, 0.0, 0.0, 0.0]), np.array([-0.1, -0.1]), np.array([0.1, 0.1]),
                          support_obb=0)]
    return s


class OracleCtx:
    """CPU stand-in for TampContext (the oracle's arithmetic; test infrastructure)."""

    def __init__(self, spec, n, device=None):
        self.spec, self.n = spec, n
        self.csp = O.build_csp(spec)
        self.n_hard = len(self.csp.terms)

    def sample(self, seed):
        x, g = O.initialize_particles(self.spec, self.csp, seed, np.arange(self.n))
        self.st = O.new_state(x, g)

    def optimize(self, k):
        O.optimize(self.spec, self.csp, self.st, k, 1.0 / self.n)

    def check(self):
        _, c, *_ = O.check(self.spec, self.csp, self.st)
        return torch.tensor(c, dtype=torch.int32), None

    def best_k(self, k):
        cls, _, J, soft, _ = O.check(self.spec, self.csp, self.st)
        sel, kc, kcost = O.best_k(cls, J, soft, np.arange(self.n), k)
        out = torch.zeros(k, self.csp.D + 4)
        out[:, 0] = torch.tensor(kc, dtype=torch.float32)
        return out


def _heuristic(counts, n_hard, penalty):
    return O.plan_heuristic(list(np.asarray(counts)[:n_hard]), penalty)


def test_algorithm1_loop_cpu(monkeypatch):
    monkeypatch.setattr(planner, "TampContext", OracleCtx)
    monkeypatch.setattr(planner, "plan_heuristic", _heuristic)
    spec = make_config(1, n=64)
    spec.ik_iters = 20
    res = planner.cutamp([_infeasible_variant(spec), spec], 64, seed=3, steps_per_pop=20, check_every=10,
                         max_pops=4, k=2)
    assert res is not None and res.skeleton == 1
    assert res.heuristics[1] > res.heuristics[0]        # the infeasible skeleton has zero-count constraints
    assert int(res.records[0, 0]) == 0                   # best record is satisfying


@pytest.mark.gpu
def test_algorithm1_loop_gpu():
    torch.cuda.set_device(0)
    spec = make_config(1, n=1024)
    spec.ik_iters = 20
    res = planner.cutamp([_infeasible_variant(spec), spec], 1024, seed=3, steps_per_pop=100, k=4)
    assert res is not None and res.skeleton == 1 and res.pops == 1
    cls, cost, gidx, x = planner.decode_records(res.records)
    assert cls[0] == 0


@pytest.mark.gpu
def test_stick_button_skeletons_gpu():
    """Stick Button: pressing the out-of-reach blue button with the fingertip never
    satisfies its Kin constraint (zero count -> Eq. 5 penalty), the stick skeleton is solved; Algorithm 1
    therefore refines the stick skeleton first and returns its satisfying particles."""
    torch.cuda.set_device(0)
    n = 4096
    direct, stick = make_config(7, n=n), make_config(6, n=n)
    for s in (direct, stick):
        s.ik_iters = 20
    ctx = planner.TampContext(direct, n)
    ctx.sample(seed=1)
    ctx.optimize(300)
    counts, _ = ctx.check()
    kp_blue = [i for i, k in enumerate(ctx.term_kinds) if k == "KP"][1]
    assert int(counts[kp_blue]) == 0 and int(counts[-2]) == 0
    res = planner.cutamp([direct, stick], n, seed=5, steps_per_pop=300, max_pops=4, k=4)
    assert res is not None and res.skeleton == 1 and res.pops == 1
    assert res.heuristics[1] > res.heuristics[0]
    cls, cost, gidx, x = planner.decode_records(res.records)
    assert cls[0] == 0
