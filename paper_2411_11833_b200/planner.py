"""Algorithm 1 (cuTAMP) over a given set of candidate plan skeletons -- SURVEY §8(f) f3.

Host-side control loop around the hot path: every skeleton's particles are initialised on the GPU
(InitializeParticles, tamp_sample_particles) and scored with the plan-feasibility heuristic
Eq. 5 from the satisfied counts of tamp_check_satisfied; a priority queue ordered by the
heuristic then repeatedly pops the most promising skeleton, optimises its particles for a step budget
(OptimizeParticles, tamp_optimize_step, checking Eq. 3 every `check_every` steps), returns the best
satisfying particles as soon as any exist and otherwise re-scores and re-pushes it
(P:349-351).  The symbolic skeleton search (SearchPlanSkeleton) is out of scope: the caller
supplies the candidate skeletons as ProblemSpecs.

Reusing samples across skeletons: every sampled variable gets a sampler stream derived from the
signature of the subgraph that produces it (object, grasp / placement occurrence, the Pick/Place/Press it
serves and that action's grasp and placement), so skeletons sharing a subgraph draw identical samples from
the counter-based Philox generator -- the "cache" costs no memory and is exact (K1 + IK are recomputed; on a
B200 that is cheaper than storing and gathering N x D floats per subgraph).
Pruning skeletons with failed subgraphs: a Kin / StablePlace / press constraint with zero
satisfying particles after sampling marks its subgraph as likely unsatisfiable; later skeletons containing
it are not sampled; every `reinit_every` pops the failed subgraphs are re-sampled with fresh seeds and the
skeletons they pruned come back once a counterexample is found.

`method` selects the paper's baselines:
  "cutamp"        InitializeParticles with the skeleton's samplers (set spec.ik_iters > 0 for the conditional
                  IK sampler), then OptimizeParticles;
  "optimization"  the same loop from the unconditioned init (uniform confs: IK disabled);
  "sampling"      no OptimizeParticles: every `check_every` "steps" the particles are re-drawn with a fresh
                  seed (K1 + K3 only, "continuously resampled without optimization").
"""
from __future__ import annotations

import dataclasses
import heapq
import zlib
from typing import Dict, List, Optional

import torch

from .tamp import TampContext, decode_records, plan_heuristic


@dataclasses.dataclass
class PlanResult:
    skeleton: int                 # index of the solved skeleton in the candidate list
    records: torch.Tensor         # best-k records [k][D + 4] (class, cost, global index, x)
    steps: int                    # optimisation steps spent on the winning skeleton
    pops: int                     # skeleton pops (Stage 2 iterations)
    heuristics: List[float]       # Stage 1 heuristic of every skeleton (nan: pruned, never sampled)
    pruned: List[int] = dataclasses.field(default_factory=list)   # skeletons still pruned at the end


METHODS = ("cutamp", "optimization", "sampling")
# action kinds (include/tamp.h)
_MOVE_FREE, _PICK, _MOVE_HOLD, _PLACE, _PRESS, _PRESS_STICK = range(6)
_VAR_CONF, _VAR_PLACEMENT, _VAR_GRASP, _VAR_TRAJ = range(4)
_LOCAL_TERMS = ("KP", "KR", "SS", "SC", "PC")     # depend only on their action's sampled subgraph


def subgraph_signatures(spec) -> Dict[int, tuple]:
    """Free variable index -> signature of the sampling subgraph that produces it."""
    V = spec.variables
    objs, surfs = spec.objects, spec.surfaces
    sig: Dict[int, tuple] = {}
    occ: Dict[tuple, int] = {}

    def nth(key):
        occ[key] = occ.get(key, -1) + 1
        return occ[key]

    def ref(vi):
        v = V[vi]
        if v.const:
            return ("const", tuple(round(float(a), 6) for a in v.value))
        return sig.get(vi, ("var", vi))

    for vi, v in enumerate(V):
        if v.const:
            continue
        if v.kind == _VAR_GRASP:
            sig[vi] = ("grasp", objs[v.obj].name, nth(("g", v.obj)))
        elif v.kind == _VAR_PLACEMENT:
            sig[vi] = ("placement", objs[v.obj].name, surfs[v.surface].name, nth(("p", v.obj, v.surface)))
    for a in spec.actions:
        if a.kind in (_PICK, _PLACE, _PRESS, _PRESS_STICK) and not V[a.q1].const:
            sig[a.q1] = ("conf", a.kind, objs[a.obj].name, ref(a.grasp), ref(a.placement))
    for vi, v in enumerate(V):
        if not v.const and v.kind == _VAR_CONF and vi not in sig:
            sig[vi] = ("conf", "free", nth(("q",)))
    for a in spec.actions:
        if a.kind in (_MOVE_FREE, _MOVE_HOLD) and a.traj >= 0:
            sig[a.traj] = ("traj", ref(a.q1), ref(a.q2), V[a.traj].n_knots)
    return sig


def with_subgraph_streams(spec):
    """Copy of spec whose sampled variables use streams keyed by their subgraph signatures."""
    sig = subgraph_signatures(spec)
    vs = [dataclasses.replace(v, rng_stream=(zlib.crc32(repr(sig[i]).encode()) | 1) if i in sig else 0)
          for i, v in enumerate(spec.variables)]
    return dataclasses.replace(spec, variables=vs)


def local_term_signatures(spec, term_kinds, term_actions) -> List[Optional[tuple]]:
    """Per hard term: a skeleton-independent signature for the Kin / StablePlace / press terms (None else)."""
    sig = subgraph_signatures(spec)
    out = []
    for kind, ai in zip(term_kinds, term_actions):
        a = spec.actions[ai] if ai >= 0 else None
        if kind not in _LOCAL_TERMS or a is None:
            out.append(None)
        elif kind in ("KP", "KR"):
            out.append((kind, sig.get(a.q1)))
        else:
            out.append((kind, sig.get(a.placement)))
    return out


def cutamp(skeletons, n_particles: int, seed: int = 0, steps_per_pop: int = 200, check_every: int = 10,
           max_pops: int = 20, k: int = 8, penalty: float = -1e6, device=None, method: str = "cutamp",
           share_samples: bool = True, prune: bool = True, reinit_every: int = 4) -> Optional[PlanResult]:
    """Solve with Algorithm 1 over the candidate skeletons (ProblemSpecs of one TAMP problem)."""
    if method not in METHODS:
        raise ValueError(f"method must be one of {METHODS}")
    n_sk = len(skeletons)
    ctxs: List = [None] * n_sk
    tsigs: List = [None] * n_sk
    h0: List[float] = [float("nan")] * n_sk
    queue: list = []
    draws = [0] * n_sk
    spent = [0] * n_sk
    failed: Dict[tuple, int] = {}      # unsatisfiable-looking subgraph -> skeleton that showed it
    pruned: List[int] = []

    def fresh_seed(i):
        draws[i] += 1
        return seed + 7919 * i + 104729 * draws[i]

    def start(i):                       # InitializeParticles + PlanHeuristic, then queue it
        ctx = ctxs[i]
        ctx.sample(seed + 7919 * i)
        counts, _ = ctx.check()
        c = counts.cpu()
        for t, sg in enumerate(tsigs[i]):
            if sg is not None and int(c[t]) == 0:
                failed.setdefault(sg, i)
        h = plan_heuristic(c, ctx.n_hard, penalty)
        h0[i] = h
        heapq.heappush(queue, (-h, i))

    for i, spec in enumerate(skeletons):           # Stage 1
        if method == "optimization" and getattr(spec, "ik_iters", 0):
            spec = dataclasses.replace(spec, ik_iters=0)
        if share_samples:
            spec = with_subgraph_streams(spec)
        ctxs[i] = TampContext(spec, n_particles, device=device)
        kinds = getattr(ctxs[i], "term_kinds", None)
        acts = getattr(ctxs[i], "term_actions", None)
        tsigs[i] = local_term_signatures(spec, kinds, acts) if kinds is not None and acts is not None \
            else [None] * ctxs[i].n_hard
        if prune and any(sg in failed for sg in tsigs[i] if sg is not None):
            pruned.append(i)                         # same failed subgraph as an earlier skeleton
            continue
        start(i)
    for pops in range(1, max_pops + 1):             # Stage 2
        if prune and failed and reinit_every > 0 and pops % reinit_every == 0:
            for sg, j in list(failed.items()):      # re-initialise the failed subgraphs
                ctx = ctxs[j]
                ctx.sample(fresh_seed(j))            # (skeleton j restarts from fresh particles ...)
                counts, _ = ctx.check()
                t = tsigs[j].index(sg)
                if int(counts[t]) > 0:               # counterexample: the subgraph is feasible
                    del failed[sg]
                # ... so its queue key is that of the fresh particles, not of the state it replaced
                queue[:] = [e for e in queue if e[1] != j]
                heapq.heapify(queue)
                h = plan_heuristic(counts.cpu(), ctx.n_hard, penalty)
                heapq.heappush(queue, (-h, j))
            for i in list(pruned):
                if not any(sg in failed for sg in tsigs[i] if sg is not None):
                    pruned.remove(i)
                    start(i)
        if not queue:
            break
        _, i = heapq.heappop(queue)
        ctx = ctxs[i]
        for _ in range(steps_per_pop // check_every):
            if method == "sampling":                 # re-draw instead of optimising
                ctx.sample(fresh_seed(i))
                counts, _ = ctx.check()              # IsGoalSatisfied (Eq. 3)
            elif hasattr(ctx, "optimize_check"):     # OptimizeParticles + IsGoalSatisfied in one launch
                counts, _ = ctx.optimize_check(check_every)
            else:
                ctx.optimize(check_every)
                counts, _ = ctx.check()
            spent[i] += check_every
            if int(counts[-2].item()) > 0:           # GetSatisfyingParticles (best first)
                return PlanResult(i, ctx.best_k(k), spent[i], pops, h0, pruned=list(pruned))
        h = plan_heuristic(counts.cpu(), ctx.n_hard, penalty)
        heapq.heappush(queue, (-h, i))               # add back to the queue with the new heuristic
    return None


__all__ = ["cutamp", "PlanResult", "decode_records", "subgraph_signatures", "with_subgraph_streams",
           "local_term_signatures", "METHODS"]
