"""Hand-constructed particles for tests (inputs only; the values they must produce are worked out in the tests).

`pickplace_hold_knots` is config 1 in an empty world (no OBBs, a 4x4 m region on z = 0) whose
MoveHold carries free knots, so a satisfying particle has a nonzero soft cost (TrajLength, Listing 1 cost)
that differs between particles: the best-k key of a satisfying particle (L19) is then exercised.
"""
import math

import numpy as np
import torch

from oracle import tamp_oracle as O
from workloads.scenes import (Action, Surface, Var, CONF, GRASP, PLACEMENT, TRAJ, MOVE_FREE, MOVE_HOLD, PICK,
                              PLACE, Q_HOME, block, _f32, _spec, _Builder, _table_bounds)


def pickplace_hold_knots(n=4, knots=2):
    objs = [block("red", 0.05, [0.45, -0.30, 0.0, 0.0])]
    surfs = [Surface("big", np.array([0.0, 0.0, 0.0, 0.0]), np.array([-2.0, -2.0]), np.array([2.0, 2.0]))]
    b = _Builder()
    q0 = b.var(Var(CONF, "q0", const=True, value=Q_HOME.copy()))
    p0 = b.var(Var(PLACEMENT, "p0_red", const=True, value=objs[0].init_pose.copy(), obj=0))
    lo, hi = _table_bounds()
    g = b.var(Var(GRASP, "g_red", obj=0))
    qa = b.var(Var(CONF, "q_pick"))
    qb = b.var(Var(CONF, "q_place"))
    p1 = b.var(Var(PLACEMENT, "p_red", obj=0, surface=0, lo=lo, hi=hi))
    t2 = b.var(Var(TRAJ, "tau_hold", n_knots=knots))
    b.actions += [Action(MOVE_FREE, q1=q0, q2=qa), Action(PICK, obj=0, grasp=g, placement=p0, q1=qa),
                  Action(MOVE_HOLD, obj=0, grasp=g, q1=qa, q2=qb, traj=t2),
                  Action(PLACE, obj=0, grasp=g, placement=p1, surface=0, q1=qb)]
    return _f32(_spec("pickplace_hold_knots", objs, [], surfs, b, [], n, 100))


def satisfying_pickplace(spec, csp, rng, psi):
    """q_pick random (joint 1 kept 0.7 rad inside its limits); T(g) := T(p0)^-1 FK(q_pick); the place
    is everything rotated by psi about the base axis: p1 = Rz(psi) p0, q_place = q_pick + psi e_1 (joint 1 is
    the world z axis through the base); knots on the straight line q_pick -> q_place.  Every hard term is 0
    up to rounding and the soft cost is lambda_traj * |psi|."""
    V = spec.variables
    vid = {v.name: i for i, v in enumerate(V)}
    rob = spec.robot
    lo, hi = rob.joint_lo.copy(), rob.joint_hi.copy()
    lo[0] += 0.7
    hi[0] -= 0.7
    q = rng.uniform(lo, hi)
    p0 = V[vid["p0_red"]].value
    F = O.forward_kinematics(rob, torch.tensor(q[None]))[0, 8]
    Tg = (O.inverse(O.pose_xyzyaw(torch.tensor(p0))) @ F).numpy()[:3]
    c, s = math.cos(psi), math.sin(psi)
    p1 = np.array([c * p0[0] - s * p0[1], s * p0[0] + c * p0[1], p0[2], p0[3] + psi])
    x = np.zeros(csp.D)
    q2 = q.copy()
    q2[0] += psi
    x[csp.offsets[vid["q_pick"]]:csp.offsets[vid["q_pick"]] + 7] = q
    x[csp.offsets[vid["q_place"]]:csp.offsets[vid["q_place"]] + 7] = q2
    x[csp.offsets[vid["p_red"]]:csp.offsets[vid["p_red"]] + 4] = p1
    K = V[vid["tau_hold"]].n_knots
    off = csp.offsets[vid["tau_hold"]]
    for j in range(K):
        x[off + 7 * j:off + 7 * j + 7] = q + (j + 1) / (K + 1) * (q2 - q)
    return x, Tg
