"""Algorithm 1 (cuTAMP) over a given set of candidate plan skeletons -- SURVEY §8(f) f3.

Host-side control loop around the hot path: every skeleton's particles are initialised on the GPU
(InitializeParticles, tamp_sample_particles) and scored with the plan-feasibility heuristic
Eq. 5 from the satisfied counts of tamp_check_satisfied; a priority queue ordered by the
heuristic then repeatedly pops the most promising skeleton, optimises its particles for a step budget
(OptimizeParticles, tamp_optimize_step, checking Eq. 3 every `check_every` steps), returns the best
satisfying particles as soon as any exist and otherwise re-scores and re-pushes it
(P:349-351).  The symbolic skeleton search (SearchPlanSkeleton) is out of scope: the caller
supplies the candidate skeletons as ProblemSpecs.  Subgraph caching is not implemented.
"""
from __future__ import annotations

import dataclasses
import heapq
from typing import List, Optional

import torch

from .tamp import TampContext, decode_records, plan_heuristic


@dataclasses.dataclass
class PlanResult:
    skeleton: int                 # index of the solved skeleton in the candidate list
    records: torch.Tensor         # best-k records [k][D + 4] (class, cost, global index, x)
    steps: int                    # optimisation steps spent on the winning skeleton
    pops: int                     # skeleton pops (Stage 2 iterations)
    heuristics: List[float]       # Stage 1 heuristic of every skeleton


def cutamp(skeletons, n_particles: int, seed: int = 0, steps_per_pop: int = 200, check_every: int = 10,
           max_pops: int = 20, k: int = 8, penalty: float = -1e6, device=None) -> Optional[PlanResult]:
    """Solve with Algorithm 1 over the candidate skeletons (ProblemSpecs of one TAMP problem)."""
    ctxs, queue, h0 = [], [], []
    for i, spec in enumerate(skeletons):           # Stage 1: InitializeParticles + PlanHeuristic
        ctx = TampContext(spec, n_particles, device=device)
        ctx.sample(seed + 7919 * i)
        counts, _ = ctx.check()
        h = plan_heuristic(counts.cpu(), ctx.n_hard, penalty)
        ctxs.append(ctx)
        h0.append(h)
        heapq.heappush(queue, (-h, i))
    spent = [0] * len(skeletons)
    for pops in range(1, max_pops + 1):             # Stage 2
        if not queue:
            break
        _, i = heapq.heappop(queue)
        ctx = ctxs[i]
        for _ in range(steps_per_pop // check_every):
            ctx.optimize(check_every)                # OptimizeParticles
            spent[i] += check_every
            counts, _ = ctx.check()                  # IsGoalSatisfied (Eq. 3)
            if int(counts[-2].item()) > 0:           # GetSatisfyingParticles (best first)
                return PlanResult(i, ctx.best_k(k), spent[i], pops, h0)
        h = plan_heuristic(counts.cpu(), ctx.n_hard, penalty)
        heapq.heappush(queue, (-h, i))               # add back to the queue with the new heuristic
    return None


__all__ = ["cutamp", "PlanResult", "decode_records"]
