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


# ---------------------------------------------------------------------------------------------------
# Tetris (configs 3 / 4): an exactly tiled satisfying particle ("feasible by construction")
# ---------------------------------------------------------------------------------------------------
def _rot_cells(cells, k):
    c = np.asarray(cells, float)
    R = np.array([[0.0, -1.0], [1.0, 0.0]])
    for _ in range(k):
        c = c @ R.T
    return c


def tile_grid(W, H, shapes):
    """Backtracking tiling of a W x H cell grid with the given tetrominoes (rotations only, no reflection).
    Returns [(k, ox, oy)] per piece: rotation by k quarter turns, then translation so the cells start at (ox, oy)."""
    from workloads.scenes import TETROMINOES
    grid = -np.ones((W, H), int)
    sol = []

    def rec(i):
        if i == len(shapes):
            return True
        for k in range(4):
            r = _rot_cells(TETROMINOES[shapes[i]], k)
            r = np.rint(r - r.min(axis=0)).astype(int)
            for ox in range(W):
                for oy in range(H):
                    c = r + [ox, oy]
                    if (c[:, 0] >= W).any() or (c[:, 1] >= H).any() or (grid[c[:, 0], c[:, 1]] >= 0).any():
                        continue
                    grid[c[:, 0], c[:, 1]] = i
                    sol.append((k, ox, oy))
                    if rec(i + 1):
                        return True
                    grid[c[:, 0], c[:, 1]] = -1
                    sol.pop()
        return False

    assert rec(0), "no tiling"
    return sol


def tetris_tiled_placements(spec, W, H, shapes):
    """Placements (x, y, z, yaw) of the pieces tiling the W x H grid centred in the goal region.  A piece's object
    frame has its cells centred on their mean (workloads.tetromino), so yaw k pi/2 maps them onto R^k c - R^k mean,
    and the centroid lands at R^k mean - min(R^k c) + offset (cell units)."""
    from workloads.scenes import TETROMINOES, CELL
    sf = [s for s in spec.surfaces if s.name == "tetris_region"][0]
    cx, cy = sf.frame[0], sf.frame[1]
    out = []
    for shape, (k, ox, oy) in zip(shapes, tile_grid(W, H, shapes)):
        c = np.asarray(TETROMINOES[shape], float)
        rc = _rot_cells(c, k)
        t = _rot_cells(c.mean(axis=0)[None], k)[0] - rc.min(axis=0) + [ox, oy]
        out.append(np.array([cx + (t[0] - (W - 1) / 2) * CELL, cy + (t[1] - (H - 1) / 2) * CELL, sf.frame[2],
                             k * math.pi / 2]))
    return out


def _ik(spec, T, rng, tries=32, iters=300, tol=(1e-7, 1e-7)):
    """Confs reaching T (errors below tol: exact by default), from random starts solved as one batch: the oracle's
    DLS IK (pinned)."""
    rob = spec.robot
    q0 = rng.uniform(rob.joint_lo, rob.joint_hi, (tries, 7))
    q = O.ik_dls(rob, q0, np.broadcast_to(T, (tries, 4, 4)).copy(), iters, 0.05)
    ep, th = O.ik_errors(rob, q, np.broadcast_to(T, (tries, 4, 4)).copy())
    for k in range(tries):
        if ep[k] < tol[0] and th[k] < tol[1]:
            yield q[k]


def satisfying_tetris(spec, csp, rng, W, H, shapes, lift=0.2, ik_tol=(1e-7, 1e-7)):
    """Hand-constructed satisfying particle of a Tetris skeleton: pieces on an exact tiling of the grid (z on the
    region, yaws multiples of pi/2), top-down grasps over each piece's centroid with the gripper turned so its
    fingers lie along the piece's own cells (searched over 24 yaws), pick / place confs by exact IK
    (T(g) := placement-consistent, FK(q) = T(p) T(g)), each chosen among IK solutions so that its own CF terms are
    exactly 0 (ik_tol: the Kin residual accepted -- exact by default; config 4's last pick is at the arm's reach,
    where 1 mm / 0.01 rad, a fifth of the 5 mm / 0.05 rad tolerances of P:1133, is what the IK attains);
    knots (config 4) at confs reaching the same TCP poses lifted by `lift`.  Every pick / place and knot
    is checked with the oracle (CF, JL; Kin by construction); returns (x [D], grasps [G, 3, 4])."""
    V = spec.variables
    vid = {v.name: i for i, v in enumerate(V)}
    x = np.zeros(csp.D)
    G = np.zeros((len(csp.grasp_vars), 3, 4))
    G[:, 0, 0] = G[:, 1, 1] = G[:, 2, 2] = 1.0
    places = tetris_tiled_placements(spec, W, H, shapes)
    names = [o.name for o in spec.objects]
    terms_of = {}
    for ti, t in enumerate(csp.terms):
        terms_of.setdefault(t.action, []).append(ti)
    eps = np.array([spec.eps[t.kind] for t in csp.terms])

    def eval_terms(tids):            # the oracle on a CSP holding only these terms (one FK per conf involved)
        import dataclasses
        sub = dataclasses.replace(csp, terms=[csp.terms[t] for t in tids], goal={}, traj_costs=[])
        with torch.no_grad():
            _, Jc, _ = O.evaluate(spec, sub, torch.as_tensor(x[None]), torch.as_tensor(G[None]))
        return Jc.numpy()[0]

    def set_conf(vi, q):
        x[csp.offsets[vi]:csp.offsets[vi] + 7] = q

    def up(T):
        T = T.copy()
        T[2, 3] += lift
        return T

    for i, nm in enumerate(names):
        # Listing 1 order per piece: MoveFree, Pick, MoveHold, Place
        ai = 4 * i
        a_pick, a_place = spec.actions[ai + 1], spec.actions[ai + 3]
        vp = a_place.placement
        x[csp.offsets[vp]:csp.offsets[vp] + 4] = places[i]
        gslot = csp.grasp_vars.index(a_pick.grasp)
        o = spec.objects[i]
        done = False
        cands = [(0.0, 0.0, gm) for gm in rng.permutation(np.arange(24) * math.pi / 12)]
        cands += [(gx, gy, gm) for gx, gy, gm in zip(rng.uniform(-o.grasp_xy, o.grasp_xy, 48),
                                                      rng.uniform(-o.grasp_xy, o.grasp_xy, 48),
                                                      rng.uniform(-math.pi, math.pi, 48))]
        for gx, gy, gamma in cands:
            Tg = O.top_down_grasp(torch.tensor([gx]), torch.tensor([gy]), torch.tensor([o.grasp_z]),
                                  torch.tensor([gamma]))[0].numpy()
            G[gslot] = Tg[:3]
            T_pick = (O.pose_xyzyaw(torch.tensor(V[a_pick.placement].value)).numpy() @ Tg)
            T_place = (O.pose_xyzyaw(torch.tensor(places[i])).numpy() @ Tg)
            ok = True
            for a_idx, T in ((ai + 1, T_pick), (ai + 3, T_place)):
                a = spec.actions[a_idx]
                good = False
                for q in _ik(spec, T, rng, tol=ik_tol):
                    set_conf(a.q1, q)
                    tids = [t for t in terms_of[a_idx] if csp.terms[t].kind in ("JL", "CF")]
                    if np.all(eval_terms(tids) == 0.0):
                        good = True
                        break
                if not good:
                    ok = False
                    break
            if ok:
                done = True
                break
        assert done, f"no collision-free grasp / IK for {nm}"
        # knots: lifted TCP poses (config 4), checked like the confs
        for a_idx in (ai, ai + 2):
            a = spec.actions[a_idx]
            if a.traj < 0 or V[a.traj].n_knots == 0:
                continue
            K = V[a.traj].n_knots
            if a_idx == ai:      # MoveFree into the pick: lifted above the pick
                poses = [up(T_pick)] * K
            else:                # MoveHold: lifted above the pick, then above the place
                poses = [up(T_pick)] + [up(T_place)] * (K - 1)
            for j, T in enumerate(poses):
                good = False
                for q in _ik(spec, T, rng):
                    x[csp.offsets[a.traj] + 7 * j:csp.offsets[a.traj] + 7 * j + 7] = q
                    tids = [t for t in terms_of[a_idx] if csp.terms[t].conf == ("knot", a.traj, j)]
                    if np.all(eval_terms(tids) == 0.0):
                        good = True
                        break
                assert good, f"no collision-free knot {j} for action {a_idx}"
    return x, G
