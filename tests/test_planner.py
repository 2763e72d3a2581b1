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
    direct2 = copy.deepcopy(direct)                      # same failed subgraph: pruned, never sampled
    res = planner.cutamp([direct, direct2, stick], n, seed=5, steps_per_pop=300, max_pops=4, k=4)
    assert res is not None and res.skeleton == 2 and res.pops == 1
    assert res.heuristics[2] > res.heuristics[0] and res.pruned == [1]
    cls, cost, gidx, x = planner.decode_records(res.records)
    assert cls[0] == 0


class _RecCtx:
    """Records the calls Algorithm 1 makes (no arithmetic)."""
    log = []

    def __init__(self, spec, n, device=None):
        self.spec, self.n, self.n_hard = spec, n, 3
        _RecCtx.log.append(("init", getattr(spec, "ik_iters", 0)))

    def sample(self, seed):
        _RecCtx.log.append(("sample", seed))

    def optimize(self, k):
        _RecCtx.log.append(("optimize", k))

    def check(self):
        return torch.tensor([1, 1, 1, 0, 0], dtype=torch.int32), None


@pytest.mark.parametrize("method", ["cutamp", "optimization", "sampling"])
def test_baseline_methods_call_pattern(monkeypatch, method):
    """f1 baselines: Optimization = uniform init (IK off) + optimise; Sampling = fresh draws, never
    optimised; cuTAMP = the skeleton's samplers (IK as configured) + optimise."""
    monkeypatch.setattr(planner, "TampContext", _RecCtx)
    _RecCtx.log = []
    spec = make_config(1, n=8)
    spec.ik_iters = 20
    res = planner.cutamp([spec], 8, seed=1, steps_per_pop=30, check_every=10, max_pops=2, method=method)
    assert res is None
    kinds = [c[0] for c in _RecCtx.log]
    assert _RecCtx.log[0] == ("init", 0 if method == "optimization" else 20)
    if method == "sampling":
        assert "optimize" not in kinds
        seeds = [c[1] for c in _RecCtx.log if c[0] == "sample"]
        assert len(seeds) == 1 + 2 * 3 and len(set(seeds)) == len(seeds)
    else:
        assert kinds.count("optimize") == 6 and kinds.count("sample") == 1
    with pytest.raises(ValueError):
        planner.cutamp([spec], 8, method="bogus")


# ---------------------------------------------------------------------------------------------
# reusing samples across skeletons and pruning failed subgraphs
# ---------------------------------------------------------------------------------------------
def _cols(spec, csp, vi):
    off = csp.offsets[vi]
    return slice(off, off + (7 if spec.variables[vi].kind == 0 else 4))


def test_shared_subgraph_draws_identical_samples():
    """Skeletons 6 and 7 share PressButton(red) (fingertip grasp, press pose, IK conf): with subgraph streams
    the oracle's InitializeParticles (incl. the conditional IK sampler) gives identical values for it; the
    unshared press poses differ; and without streams the shared subgraph is drawn independently."""
    a, b = make_config(6, n=16), make_config(7, n=16)
    for s in (a, b):
        s.ik_iters = 5
    sa, sb = planner.with_subgraph_streams(a), planner.with_subgraph_streams(b)
    ca, cb = O.build_csp(sa), O.build_csp(sb)
    xa, ga = O.initialize_particles(sa, ca, 9, np.arange(16))
    xb, gb = O.initialize_particles(sb, cb, 9, np.arange(16))
    name = {v.name: i for i, v in enumerate(a.variables)}
    nameb = {v.name: i for i, v in enumerate(b.variables)}
    for v in ("press_red", "q_press_red"):
        np.testing.assert_array_equal(xa[:, _cols(a, ca, name[v])], xb[:, _cols(b, cb, nameb[v])])
    np.testing.assert_array_equal(ga[:, ca.grasp_vars.index(name["g_fingertip"])],
                                  gb[:, cb.grasp_vars.index(nameb["g_fingertip"])])
    assert not np.array_equal(xa[:, _cols(a, ca, name["q_press_blue"])], xb[:, _cols(b, cb, nameb["q_press_blue"])])
    # default streams (variable indices): the same subgraph is sampled independently
    x0, _ = O.initialize_particles(a, O.build_csp(a), 9, np.arange(16))
    assert not np.array_equal(x0[:, _cols(a, ca, name["press_red"])], xa[:, _cols(a, ca, name["press_red"])])
    sig = planner.subgraph_signatures(a)
    assert len({sig[i] for i in sig}) == len(sig)                       # distinct subgraphs, distinct streams


class _PruneCtx:
    """Oracle-backed context (term structure from the oracle's build_csp) with counts from the oracle's check."""
    sampled = []

    def __init__(self, spec, n, device=None):
        self.spec, self.n = spec, n
        self.csp = O.build_csp(spec)
        self.n_hard = len(self.csp.terms)
        self.term_kinds = [t.kind for t in self.csp.terms]
        self.term_actions = [t.action for t in self.csp.terms]

    def sample(self, seed):
        _PruneCtx.sampled.append(self.spec.name)
        x, g = O.initialize_particles(self.spec, self.csp, seed, np.arange(self.n))
        self.st = O.new_state(x, g)

    def optimize(self, k):
        O.optimize(self.spec, self.csp, self.st, k, 1.0 / self.n)

    def check(self):
        _, c, *_ = O.check(self.spec, self.csp, self.st)
        return torch.tensor(c, dtype=torch.int32), None

    def best_k(self, k):
        return torch.zeros(k, self.csp.D + 4)


def test_failed_subgraph_prunes_later_skeletons(monkeypatch):
    """Pressing the out-of-reach blue button with the fingertip has zero Kin-satisfying particles after
    sampling; a later skeleton containing the same press subgraph is pruned (never sampled) and
    stays pruned through the periodic re-initialisation; the stick skeleton is sampled and queued."""
    monkeypatch.setattr(planner, "TampContext", _PruneCtx)
    monkeypatch.setattr(planner, "plan_heuristic", _heuristic)
    _PruneCtx.sampled = []
    direct = make_config(7, n=32)
    direct2 = copy.deepcopy(direct)
    direct2.name = "direct_again"
    stick = make_config(6, n=32)
    for s in (direct, direct2, stick):
        s.ik_iters = 10
    res = planner.cutamp([direct, direct2, stick], 32, seed=2, steps_per_pop=10, check_every=10, max_pops=4,
                         reinit_every=2)
    assert "direct_again" not in _PruneCtx.sampled and "stickbutton" in _PruneCtx.sampled
    assert _PruneCtx.sampled.count("stickbutton_direct") >= 2          # initial draw + re-initialisations
    assert res is None or res.skeleton != 1
    sig = planner.local_term_signatures(planner.with_subgraph_streams(direct), *(
        lambda c: ([t.kind for t in c.terms], [t.action for t in c.terms]))(O.build_csp(direct)))
    kp_blue = [s for s, k in zip(sig, [t.kind for t in O.build_csp(direct).terms]) if k == "KP"][1]
    assert kp_blue[1][1] == 4 and kp_blue[1][2] == "fingertip"        # (KP, conf of PressButton(fingertip))


def test_reinit_requeues_the_reset_skeleton(monkeypatch):
    """Re-initialising a failed subgraph re-samples its skeleton's whole context, so the skeleton must be queued
    again with the heuristic of the fresh particles -- every sampling of a skeleton is followed by a push of that
    skeleton, and the queue never holds two entries of one skeleton (planner.py)."""
    events = []

    class Ctx(_PruneCtx):
        def sample(self, seed):
            events.append(("sample", self.spec.name))
            super().sample(seed)

    monkeypatch.setattr(planner, "TampContext", Ctx)
    monkeypatch.setattr(planner, "plan_heuristic", _heuristic)
    real_push = planner.heapq.heappush
    names = {}

    def push(q, e):
        assert e[1] not in [x[1] for x in q]
        events.append(("push", names[e[1]]))
        real_push(q, e)
    monkeypatch.setattr(planner.heapq, "heappush", push)
    _PruneCtx.sampled = []
    direct = make_config(7, n=32)
    stick = make_config(6, n=32)
    for s_ in (direct, stick):
        s_.ik_iters = 10
    names.update({0: direct.name, 1: stick.name})
    planner.cutamp([direct, stick], 32, seed=2, steps_per_pop=10, check_every=10, max_pops=3, reinit_every=2)
    samples = [k for k, e in enumerate(events) if e == ("sample", direct.name)]
    assert len(samples) >= 2                                   # the initial draw + a re-initialisation
    for k in samples:
        assert ("push", direct.name) in events[k + 1:k + 2]
