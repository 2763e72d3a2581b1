"""Float64 CPU oracle for the cuTAMP particle-optimisation hot path (TEST INFRASTRUCTURE ONLY).

Follows PAPER.md in the paper's own order and notation:
  * skeleton -> constraint set con(pi) and costs cost(pi)          (Listing 1)
  * particle x = assignment to the free continuous variables
  * J(x) = sum_c lambda_c J_c + sum_c' lambda_c' c'   (Eq. 2)
  * satisfied iff AND_c J_c <= eps_c                  (Eq. 3)
  * J_batch = 1/N sum_x J(x), gradients, Adam         (Eq. 4)
  * InitializeParticles by composed samplers
Readings where the paper is silent are SURVEY.md §8(c) L1-L25 (listed in DESIGN.md).

Implementation style: vectorised over particles with plain PyTorch CPU ops in float64, 4x4
homogeneous transforms ("b *h 4 4", Listing 2), gradients by torch autograd (reverse
mode AD of the definition -- independent of the CUDA path's hand-derived backward).
Pins: tests/test_oracle_*.py (listed in DESIGN.md §6).  Every part of the term assembly has a closed-form pin;
tools/oracle_mutants.py applies one-line mutants (SC shrink signs, TrajLength endpoints, lambda_goal, held-object
attachment, sphere->link index, CP support exclusions) and each one fails a pin.  Parity unpinned: none.
TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this module; the product path (paper_2411_11833_b200/) never does.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional, Tuple

import numpy as np
import torch

from workloads.scenes import (ProblemSpec, CONF, PLACEMENT, GRASP, TRAJ,
                              MOVE_FREE, PICK, MOVE_HOLD, PLACE, PRESS, PRESS_STICK)
from .philox import uniforms

DT = torch.float64
HARD_KINDS = ("JL", "CF", "KP", "KR", "SS", "SC", "CP", "SELF")


# ----------------------------------------------------------------------------------------------
# Geometry on 4x4 homogeneous transforms
# ----------------------------------------------------------------------------------------------
def _t(v):
    return torch.as_tensor(v, dtype=DT)


def rot_x(a):
    """Rx(a) as [..., 4, 4]."""
    a = _t(a)
    c, s = torch.cos(a), torch.sin(a)
    z, o = torch.zeros_like(a), torch.ones_like(a)
    return torch.stack([torch.stack([o, z, z, z], -1), torch.stack([z, c, -s, z], -1),
                        torch.stack([z, s, c, z], -1), torch.stack([z, z, z, o], -1)], -2)


def rot_z(a):
    """Rz(a) as [..., 4, 4]."""
    a = _t(a)
    c, s = torch.cos(a), torch.sin(a)
    z, o = torch.zeros_like(a), torch.ones_like(a)
    return torch.stack([torch.stack([c, -s, z, z], -1), torch.stack([s, c, z, z], -1),
                        torch.stack([z, z, o, z], -1), torch.stack([z, z, z, o], -1)], -2)


def rot_y(a):
    """Ry(a) as [..., 4, 4]."""
    a = _t(a)
    c, s = torch.cos(a), torch.sin(a)
    z, o = torch.zeros_like(a), torch.ones_like(a)
    return torch.stack([torch.stack([c, z, s, z], -1), torch.stack([z, o, z, z], -1),
                        torch.stack([-s, z, c, z], -1), torch.stack([z, z, z, o], -1)], -2)


def trans(x, y, z):
    """Translation as [..., 4, 4]."""
    x, y, z = _t(x), _t(y), _t(z)
    x, y, z = torch.broadcast_tensors(x, y, z)
    zz, o = torch.zeros_like(x), torch.ones_like(x)
    return torch.stack([torch.stack([o, zz, zz, x], -1), torch.stack([zz, o, zz, y], -1),
                        torch.stack([zz, zz, o, z], -1), torch.stack([zz, zz, zz, o], -1)], -2)


def pose_xyzyaw(p):
    """Placement / 4-DOF pose (x, y, z, yaw) -> Trans(x, y, z) Rz(yaw)."""
    p = _t(p)
    return trans(p[..., 0], p[..., 1], p[..., 2]) @ rot_z(p[..., 3])


def transform_points(T, c):
    """T [..., 4, 4] applied to points c [..., M, 3] (broadcast) -> [..., M, 3]."""
    return (T[..., None, :3, :3] @ c[..., None]).squeeze(-1) + T[..., None, :3, 3]


def inverse(T):
    R = T[..., :3, :3]
    t = T[..., :3, 3]
    Ri = R.transpose(-1, -2)
    out = torch.zeros_like(T)
    out[..., :3, :3] = Ri
    out[..., :3, 3] = -(Ri @ t[..., None]).squeeze(-1)
    out[..., 3, 3] = 1.0
    return out


def forward_kinematics(robot, q):
    """Serial-chain FK ("FK(q)"): T_j = T_{j-1} Rx(alpha) Tx(a) Tz(d) Rz(q_j).

    q: [N, 7].  Returns (frames [N, 9, 4, 4] with frames[:, 0] = base, frames[:, j] = link j,
    frames[:, 8] = tool/TCP frame).
    """
    N = q.shape[0]
    base = pose_xyzyaw(robot.base).expand(N, 4, 4)
    frames = [base]
    T = base
    for j in range(7):
        a, d, alpha = (float(v) for v in robot.dh[j])
        F = rot_x(alpha) @ trans(a, 0.0, 0.0) @ trans(0.0, 0.0, d)
        T = T @ F @ rot_z(q[:, j])
        frames.append(T)
    tool = trans(0.0, 0.0, robot.flange_d) @ rot_z(robot.tcp_yaw) @ trans(0.0, 0.0, robot.tcp_d)
    frames.append(T @ tool)
    return torch.stack(frames, 1)


def robot_sphere_centers(robot, frames):
    """World centres of the robot's collision spheres: w_s = T_link(s) c_s.  [N, S, 3]."""
    c = _t(robot.spheres[:, :3])
    T = frames[:, torch.as_tensor(robot.sphere_link, dtype=torch.long)]       # [N, S, 4, 4]
    return (T[..., :3, :3] @ c[None, :, :, None]).squeeze(-1) + T[..., :3, 3]


def box_signed_distance(w, center, R, half):
    """Signed distance of points w [..., 3] to an oriented box (negative inside).

    Plain definition: p = R^T (w - c); d = |p| - h; sd = ||max(d, 0)|| + min(max_k d_k, 0).
    """
    p = (w - center) @ R          # row-vector form of R^T (w - c)
    d = p.abs() - half
    outside = torch.linalg.vector_norm(d.clamp(min=0.0), dim=-1)
    inside = d.max(dim=-1).values.clamp(max=0.0)
    return outside + inside


def obb_arrays(obb):
    """Centre, box-to-world rotation and half extents of an oriented box: the full rotation R if the
    scene gives one, else Rz(yaw) about the world z axis."""
    if getattr(obb, "R", None) is not None:
        return _t(obb.center), _t(np.asarray(obb.R, float)), _t(obb.half)
    c, s = math.cos(obb.yaw), math.sin(obb.yaw)
    R = _t([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])
    return _t(obb.center), R, _t(obb.half)


def collision_cost(p, eta, smooth=False):
    """Cost of a penetration depth p = r + eta - sd.  Hinge max(0, p) (L1); with `smooth` the CHOMP obstacle
    cost (Zucker et al. 2013; the "smooth gradients" of P:490): p - eta/2 for p > eta,
    p^2 / (2 eta) for 0 < p <= eta, 0 otherwise (continuously differentiable; needs eta > 0)."""
    if not smooth:
        return p.clamp(min=0.0)
    return torch.where(p > eta, p - eta / 2, torch.where(p > 0, p * p / (2 * eta), torch.zeros_like(p)))


def sphere_obb_cost(w, r, obbs, eta, smooth=False):
    """Sum over (sphere, box) pairs of max(0, r + eta - sd)  (L1 hinge, L2 sum)."""
    tot = torch.zeros(w.shape[0], dtype=DT)
    for obb in obbs:
        c, R, h = obb_arrays(obb)
        sd = box_signed_distance(w, c, R, h)
        tot = tot + collision_cost(r + eta - sd, eta, smooth).sum(-1)
    return tot


def sphere_sphere_cost(wa, ra, wb, rb, eta, smooth=False):
    """Sum over sphere pairs of max(0, ra + rb + eta - ||wa - wb||)."""
    d = torch.linalg.vector_norm(wa[:, :, None, :] - wb[:, None, :, :], dim=-1)
    return collision_cost(ra[:, None] + rb[None, :] + eta - d, eta, smooth).sum((-1, -2))


def dist_from_bounds(vals, lower, upper):
    """Listing 2: norm of max(lower - v, v - upper) clamped at 0."""
    diff_lower = lower - vals
    diff_upper = vals - upper
    diff_max = torch.maximum(diff_lower, diff_upper).clamp(min=0.0)
    return torch.linalg.vector_norm(diff_max, dim=-1)


def obj_dist(P):
    """Listing 2: sum over unordered pairs i<j of ||P_i - P_j||.  P [N, n, 3]."""
    n = P.shape[1]
    tot = torch.zeros(P.shape[0], dtype=DT)
    for i in range(n):
        for j in range(i + 1, n):
            tot = tot + torch.linalg.vector_norm(P[:, i] - P[:, j], dim=-1)
    return tot


def rotation_angle(Ra, Rb):
    """Geodesic angle between rotations (L4): M = Ra^T Rb, theta = atan2(||vee(M - M^T)||/2, (tr M - 1)/2)."""
    M = Ra.transpose(-1, -2) @ Rb
    w = torch.stack([M[..., 2, 1] - M[..., 1, 2], M[..., 0, 2] - M[..., 2, 0], M[..., 1, 0] - M[..., 0, 1]], -1)
    s = torch.linalg.vector_norm(w, dim=-1) / 2
    c = (M[..., 0, 0] + M[..., 1, 1] + M[..., 2, 2] - 1) / 2
    return torch.atan2(s, c)


def pose_error(Ta, Tb):
    """Kin residuals (Listing 2 curobo_pose_error P:1570-1589): (||t_a - t_b||, angle(R_a, R_b)) (L4, L5)."""
    return (torch.linalg.vector_norm(Ta[..., :3, 3] - Tb[..., :3, 3], dim=-1),
            rotation_angle(Ta[..., :3, :3], Tb[..., :3, :3]))


def six_dof_grasp(face, gx, gy, gz, gamma):
    """6-DOF grasp ("top-down 4-DOF or 6-DOF poses", PROPOSAL): face 0 = top-down as above;
    faces 1-4 approach the object's +x, -x, +y, -y side horizontally at height gz through its vertical axis:
    T(g) = Trans(0, 0, gz) R_face Rz(gamma), R_face turning the approach (TCP z) axis to -n_face."""
    top = top_down_grasp(gx, gy, gz, gamma)
    zero = torch.zeros_like(_t(gamma))
    faces = [None, rot_y(zero - math.pi / 2), rot_y(zero + math.pi / 2), rot_x(zero + math.pi / 2),
             rot_x(zero - math.pi / 2)]
    side = [None] + [trans(zero, zero, gz) @ Rf @ rot_z(gamma) for Rf in faces[1:]]
    face = torch.as_tensor(face)
    out = top.clone()
    for f in range(1, 5):
        out = torch.where((face == f)[:, None, None], side[f], out)
    return out


def top_down_grasp(gx, gy, gz, gamma):
    """Top-down 4-DOF grasp in the object frame: T(g) = Trans(gx, gy, gz) Rz(gamma) Rx(pi)  (L14)."""
    return trans(gx, gy, gz) @ rot_z(gamma) @ rot_x(torch.full_like(_t(gamma), math.pi))


# ----------------------------------------------------------------------------------------------
# Skeleton -> CSP.  The oracle's own interpretation of Listing 1 in deferred-motion mode
# plus knots when a motion carries a trajectory variable.
# ----------------------------------------------------------------------------------------------
@dataclasses.dataclass
class Term:
    kind: str                       # JL CF KP KR SS SC CP SELF PC
    conf: Optional[tuple] = None    # ("var", v) or ("knot", traj_var, j)
    scene: Optional[Dict[int, int]] = None   # object -> pose variable, objects present (not held)
    excl: Tuple[int, ...] = ()      # objects excluded from the robot check
    excl_obb: Tuple[int, ...] = ()  # OBBs excluded from the robot check (the button being pressed)
    held: Optional[Tuple[int, int]] = None   # (obj, grasp var) attached at a knot (MoveHold)
    obj: int = -1
    grasp: int = -1
    placement: int = -1
    surface: int = -1
    action: int = -1                # index of the skeleton action that emitted the term


@dataclasses.dataclass
class CSP:
    terms: List[Term]
    traj_costs: List[Tuple[int, int, int]]     # (q1 var, traj var, q2 var)
    goal: Dict[int, int]                       # goal object -> final pose var
    offsets: Dict[int, int]                    # free var -> offset in x
    D: int
    grasp_vars: List[int]
    lo: np.ndarray
    hi: np.ndarray
    lr: np.ndarray


def build_csp(spec: ProblemSpec) -> CSP:
    V = spec.variables
    # particle layout: free variables in declaration order (grasps are sampled and fixed)
    offsets, lo, hi, lr = {}, [], [], []
    D = 0
    for vi, v in enumerate(V):
        if v.const or v.kind == GRASP:
            continue
        offsets[vi] = D
        if v.kind == CONF:
            D += 7
            lo += list(spec.robot.joint_lo); hi += list(spec.robot.joint_hi); lr += [spec.lr_conf] * 7
        elif v.kind == PLACEMENT:
            D += 4
            lo += list(v.lo); hi += list(v.hi); lr += [spec.lr_pos] * 3 + [spec.lr_yaw]
        elif v.kind == TRAJ:
            D += 7 * v.n_knots
            for _ in range(v.n_knots):
                lo += list(spec.robot.joint_lo); hi += list(spec.robot.joint_hi); lr += [spec.lr_knot] * 7
    grasp_vars = [vi for vi, v in enumerate(V) if v.kind == GRASP]

    # symbolic state simulation along the skeleton (Listing 1 eff lists)
    pose = {}
    for vi, v in enumerate(V):
        if v.kind == PLACEMENT and v.const:
            pose[v.obj] = vi
    held = None
    terms: List[Term] = []
    trajs = []
    for ai, a in enumerate(spec.actions):
        n_before = len(terms)
        if a.kind in (MOVE_FREE, MOVE_HOLD):
            if a.traj >= 0 and V[a.traj].n_knots > 0:
                hv = (a.obj, a.grasp) if a.kind == MOVE_HOLD else None
                scene = {o: p for o, p in pose.items()}
                for j in range(V[a.traj].n_knots):
                    # Motion(q1, tau, q2): knots within joint limits; CFreeTraj / CFreeTrajHold at knots
                    terms.append(Term("JL", conf=("knot", a.traj, j)))
                    terms.append(Term("CF", conf=("knot", a.traj, j), scene=scene,
                                      excl=((a.obj,) if hv else ()), held=hv))
                    if spec.self_collision:   # "... does not cause robot self-collisions"
                        terms.append(Term("SELF", conf=("knot", a.traj, j)))
                trajs.append((a.q1, a.traj, a.q2))
        elif a.kind == PICK:
            scene = {o: p for o, p in pose.items()}
            c = ("var", a.q1)
            # Motion endpoint (JL), CFreeTraj endpoint + CFreeHold(o, g, q) (CF, o excluded, L3),
            # Kin(q, o, g, p) (KP, KR)
            terms.append(Term("JL", conf=c))
            terms.append(Term("CF", conf=c, scene=scene, excl=(a.obj,)))
            if spec.self_collision:
                terms.append(Term("SELF", conf=c))
            terms.append(Term("KP", conf=c, obj=a.obj, grasp=a.grasp, placement=a.placement))
            terms.append(Term("KR", conf=c, obj=a.obj, grasp=a.grasp, placement=a.placement))
            held = (a.obj, a.grasp)
            del pose[a.obj]
        elif a.kind == PLACE:
            scene = {o: p for o, p in pose.items()}
            c = ("var", a.q1)
            terms.append(Term("JL", conf=c))
            terms.append(Term("CF", conf=c, scene=scene, excl=(a.obj,)))
            if spec.self_collision:
                terms.append(Term("SELF", conf=c))
            terms.append(Term("KP", conf=c, obj=a.obj, grasp=a.grasp, placement=a.placement))
            terms.append(Term("KR", conf=c, obj=a.obj, grasp=a.grasp, placement=a.placement))
            # StablePlace(o, p, s): support + containment; CFreePlace(o, p)
            terms.append(Term("SS", obj=a.obj, placement=a.placement, surface=a.surface))
            terms.append(Term("SC", obj=a.obj, placement=a.placement, surface=a.surface))
            terms.append(Term("CP", obj=a.obj, placement=a.placement, surface=a.surface, scene=scene))
            pose[a.obj] = a.placement
            held = None
        elif a.kind in (PRESS, PRESS_STICK):
            # PressButton(b, p, q): con Kin(q, b, p), ValidPress(b, p, q); pre HandEmpty.
            # PressButtonStick(b, o, g, p, q): con Kin(q, o, g, p), ValidStickPress(o, g, p, b); pre
            # Holding(o, g).  Kin targets T(p) T(g) with p the pose of the pressing object
            # (fingertip / stick); ValidPress = the object's bottom at the face height (SS) + some sphere of
            # it over the face (PC); the held stick is also CFreePlace-checked at p except against the
            # button (CP).  The robot's CF at q ignores the button (it touches it).  DESIGN.md R8.
            s_ = spec.surfaces[a.surface]
            scene = {o: p for o, p in pose.items()}
            c = ("var", a.q1)
            btn = (s_.support_obb,) if s_.support_obb >= 0 else ()
            terms.append(Term("JL", conf=c))
            terms.append(Term("CF", conf=c, scene=scene, excl=(a.obj,), excl_obb=btn))
            if spec.self_collision:
                terms.append(Term("SELF", conf=c))
            terms.append(Term("KP", conf=c, obj=a.obj, grasp=a.grasp, placement=a.placement))
            terms.append(Term("KR", conf=c, obj=a.obj, grasp=a.grasp, placement=a.placement))
            terms.append(Term("SS", obj=a.obj, placement=a.placement, surface=a.surface))
            terms.append(Term("PC", obj=a.obj, placement=a.placement, surface=a.surface))
            if a.kind == PRESS_STICK:
                terms.append(Term("CP", obj=a.obj, placement=a.placement, surface=a.surface, scene=scene))
        for t in terms[n_before:]:
            t.action = ai
    goal = {o: pose[o] for o in spec.goal_objs}
    return CSP(terms=terms, traj_costs=trajs, goal=goal, offsets=offsets, D=D, grasp_vars=grasp_vars,
               lo=np.array(lo, float), hi=np.array(hi, float), lr=np.array(lr, float))


# ----------------------------------------------------------------------------------------------
# Particle initialisation (Algorithm 1 InitializeParticles).  Philox counter RNG.
# ----------------------------------------------------------------------------------------------
def ik_dls(robot, q, T_target, iters, damping):
    """Conditional IK sampler: damped-least-squares iterations on FK(q) = T_target.

    Per iteration (Wampler / Nakamura DLS): e = [t* - t_ee ; rotvec(R* R_ee^T)] (world frame),
    J = [z_j x (t_ee - o_j) ; z_j]_{j=1..7}, dq = J^T (J J^T + damping^2 I)^-1 e, q <- clamp(q + dq).
    q [N, 7] float64 (start: the uniform sample), T_target [N, 4, 4].
    """
    q = q.copy()
    lo, hi = robot.joint_lo, robot.joint_hi
    Tt = torch.as_tensor(T_target, dtype=DT)
    for _ in range(iters):
        F = forward_kinematics(robot, torch.as_tensor(q, dtype=DT))
        Tee = F[:, 8]
        p = Tee[:, :3, 3]
        e_p = Tt[:, :3, 3] - p
        E = Tt[:, :3, :3] @ Tee[:, :3, :3].transpose(-1, -2)
        w = torch.stack([E[:, 2, 1] - E[:, 1, 2], E[:, 0, 2] - E[:, 2, 0], E[:, 1, 0] - E[:, 0, 1]], -1)
        wn = torch.linalg.vector_norm(w, dim=-1)
        th = torch.atan2(wn / 2, (E[:, 0, 0] + E[:, 1, 1] + E[:, 2, 2] - 1) / 2)
        e_r = torch.where(wn[:, None] > 0, w * (th / torch.where(wn > 0, wn, 1.0))[:, None], torch.zeros_like(w))
        e = torch.cat([e_p, e_r], -1)                                  # [N, 6]
        cols = []
        for j in range(1, 8):
            z = F[:, j, :3, 2]
            o = F[:, j, :3, 3]
            cols.append(torch.cat([torch.linalg.cross(z, p - o), z], -1))
        J = torch.stack(cols, -1)                                      # [N, 6, 7]
        A = J @ J.transpose(-1, -2) + damping ** 2 * torch.eye(6, dtype=DT)
        y = torch.linalg.solve(A, e[..., None])
        dq = (J.transpose(-1, -2) @ y)[..., 0]
        q = np.minimum(np.maximum(q + dq.numpy(), lo), hi)
    return q


IK_TOL_POS, IK_TOL_ROT = 1e-3, 1e-3


def ik_errors(robot, q, T_target):
    """Kin errors of the tool frame at q against T_target: (||t* - t_ee||, geodesic angle of R* R_ee^T)."""
    Tee = forward_kinematics(robot, torch.as_tensor(q, dtype=DT))[:, 8]
    Tt = torch.as_tensor(T_target, dtype=DT)
    ep = torch.linalg.vector_norm(Tt[:, :3, 3] - Tee[:, :3, 3], dim=-1)
    th = rotation_angle(Tt[:, :3, :3], Tee[:, :3, :3])
    return ep.numpy(), th.numpy()


def ik_restarts(spec, q0, T_target, seed, gidx, stream):
    """The conditional IK sampler with spec.ik_seeds restarts (R6; cuRobo's solver is multi-seed,
    P:521).  Restart 0 starts from q0 (the uniform conf sample), restart s >= 1 from a fresh uniform conf drawn
    from Philox blocks 2s, 2s+1 of the conf's stream; each runs ik_dls.  Kept per particle: the first restart
    whose final errors are <= (1e-3 m, 1e-3 rad), else the one with the smallest e_pos + theta (lowest index
    on ties)."""
    S = int(getattr(spec, "ik_seeds", 1) or 1)
    lo, hi = spec.robot.joint_lo, spec.robot.joint_hi
    if S == 1:
        return ik_dls(spec.robot, q0, T_target, spec.ik_iters, spec.ik_damping)
    u = uniforms(seed, gidx, stream, 8 * S)
    qs, conv, score = [], [], []
    for s in range(S):
        start = q0 if s == 0 else lo + u[:, 8 * s:8 * s + 7] * (hi - lo)
        q = ik_dls(spec.robot, start, T_target, spec.ik_iters, spec.ik_damping)
        ep, th = ik_errors(spec.robot, q, T_target)
        qs.append(q)
        conv.append((ep <= IK_TOL_POS) & (th <= IK_TOL_ROT))
        score.append(ep + th)
    conv, score = np.stack(conv, 1), np.stack(score, 1)
    keep = np.where(conv.any(axis=1), np.argmax(conv, axis=1), np.argmin(score, axis=1))
    return np.stack(qs, 1)[np.arange(len(q0)), keep]


def _stream(V, vi):
    """Philox counter word of variable vi's sampler: its rng_stream if set, else its index."""
    return int(getattr(V[vi], "rng_stream", 0)) or vi


def initialize_particles(spec: ProblemSpec, csp: CSP, seed: int, gidx: np.ndarray):
    """Returns x0 [N, D] float64 and grasps [N, G, 3, 4] float64.

    Samplers composed in DAG order: grasps (frozen) -> placements (uniform on the surface
    region) -> confs (uniform within joint limits = the `Optimization` init; then, if
    spec.ik_iters > 0, the conditional IK sampler of P:521 toward each Pick/Place conf's Kin target
    T(p) T(g)) -> knots (linear interpolation).
    """
    V = spec.variables
    N = len(gidx)
    x = np.zeros((N, csp.D))
    grasps = np.zeros((N, len(csp.grasp_vars), 3, 4))
    for gi, vi in enumerate(csp.grasp_vars):
        o = spec.objects[V[vi].obj]
        o = dataclasses.replace(o, grasp_y=o.grasp_xy if getattr(o, "grasp_y", -1.0) < 0 else o.grasp_y)
        if getattr(o, "grasp_mode", 0) == 1:     # 6-DOF: face, gx, gy, gamma
            u = uniforms(seed, gidx, _stream(V, vi), 4)
            face = np.minimum(np.floor(u[:, 0] * 5), 4).astype(np.int64)
            gx = -o.grasp_xy + 2 * o.grasp_xy * u[:, 1]
            gy = -o.grasp_y + 2 * o.grasp_y * u[:, 2]
            gamma = -math.pi + 2 * math.pi * u[:, 3]
            T = six_dof_grasp(face, torch.as_tensor(gx), torch.as_tensor(gy),
                              torch.full((N,), o.grasp_z, dtype=DT), torch.as_tensor(gamma))
            grasps[:, gi] = T[:, :3, :].numpy()
            continue
        u = uniforms(seed, gidx, _stream(V, vi), 3)
        gx = -o.grasp_xy + 2 * o.grasp_xy * u[:, 0]
        gy = -o.grasp_y + 2 * o.grasp_y * u[:, 1]
        gamma = -math.pi + 2 * math.pi * u[:, 2]
        T = top_down_grasp(torch.as_tensor(gx), torch.as_tensor(gy), torch.full((N,), o.grasp_z, dtype=DT),
                           torch.as_tensor(gamma))
        grasps[:, gi] = T[:, :3, :].numpy()
    for vi, v in enumerate(V):
        if v.const or vi not in csp.offsets:
            continue
        off = csp.offsets[vi]
        if v.kind == CONF:
            u = uniforms(seed, gidx, _stream(V, vi), 7)
            x[:, off:off + 7] = spec.robot.joint_lo + u * (spec.robot.joint_hi - spec.robot.joint_lo)
        elif v.kind == PLACEMENT:
            s = spec.surfaces[v.surface]
            f = spec.objects[v.obj].footprint
            if any(a.kind in (PRESS, PRESS_STICK) and a.placement == vi for a in spec.actions):
                f = 0.0     # press pose: uniform on the whole button face (R8)
            u = uniforms(seed, gidx, _stream(V, vi), 3)
            wx = max(s.hi[0] - s.lo[0] - 2 * f, 0.0)
            wy = max(s.hi[1] - s.lo[1] - 2 * f, 0.0)
            lx = (s.lo[0] + s.hi[0]) / 2 - wx / 2 + u[:, 0] * wx
            ly = (s.lo[1] + s.hi[1]) / 2 - wy / 2 + u[:, 1] * wy
            lyaw = -math.pi + 2 * math.pi * u[:, 2]
            c, sn = math.cos(s.frame[3]), math.sin(s.frame[3])
            x[:, off + 0] = s.frame[0] + c * lx - sn * ly
            x[:, off + 1] = s.frame[1] + sn * lx + c * ly
            x[:, off + 2] = s.frame[2]
            x[:, off + 3] = s.frame[3] + lyaw
    if getattr(spec, "ik_iters", 0) > 0:
        gslot = {vi: k for k, vi in enumerate(csp.grasp_vars)}
        bottom = np.zeros((N, 1, 4))
        bottom[..., 3] = 1.0
        for a in spec.actions:
            if a.kind not in (PICK, PLACE, PRESS, PRESS_STICK) or V[a.q1].const:
                continue
            pv = V[a.placement]
            pval = np.broadcast_to(np.asarray(pv.value, float), (N, 4)) if pv.const else \
                x[:, csp.offsets[a.placement]:csp.offsets[a.placement] + 4]
            Tg = np.concatenate([grasps[:, gslot[a.grasp]], bottom], 1)
            Tt = (pose_xyzyaw(torch.as_tensor(np.array(pval))) @ torch.as_tensor(Tg)).numpy()
            off = csp.offsets[a.q1]
            x[:, off:off + 7] = ik_restarts(spec, x[:, off:off + 7], Tt, seed, gidx, _stream(V, a.q1))
    for a in spec.actions:
        if a.kind in (MOVE_FREE, MOVE_HOLD) and a.traj >= 0 and V[a.traj].n_knots > 0:
            K = V[a.traj].n_knots
            qa = _conf_value(spec, csp, x, a.q1)
            qb = _conf_value(spec, csp, x, a.q2)
            off = csp.offsets[a.traj]
            for j in range(K):
                x[:, off + 7 * j: off + 7 * j + 7] = qa + (j + 1) / (K + 1) * (qb - qa)
    return x, grasps


def _conf_value(spec, csp, x, vi):
    v = spec.variables[vi]
    if v.const:
        return np.broadcast_to(np.asarray(v.value, float), (x.shape[0], 7))
    return x[:, csp.offsets[vi]:csp.offsets[vi] + 7]


# ----------------------------------------------------------------------------------------------
# Eq. 2: per-particle cost, per-constraint residuals J_c and soft costs
# ----------------------------------------------------------------------------------------------
def evaluate(spec: ProblemSpec, csp: CSP, x: torch.Tensor, grasps: torch.Tensor):
    """x [N, D] (float64, may require grad), grasps [N, G, 3, 4].

    Returns (J [N], Jc [N, n_terms], soft [N]).
    """
    V = spec.variables
    rob = spec.robot
    N = x.shape[0]
    eta = spec.eta
    smooth = bool(getattr(spec, "collision_smooth", False))
    bottom = torch.zeros(1, 1, 1, 4, dtype=DT)
    bottom[..., 3] = 1.0
    G = torch.cat([grasps, bottom.expand(N, grasps.shape[1], 1, 4)], dim=-2)   # [N, G, 4, 4]
    gslot = {vi: k for k, vi in enumerate(csp.grasp_vars)}

    def var_value(vi):
        v = V[vi]
        if v.const:
            return _t(v.value).expand(N, len(v.value))
        off = csp.offsets[vi]
        return x[:, off:off + (7 if v.kind == CONF else 4)]

    def conf(c):
        if c[0] == "var":
            return var_value(c[1])
        _, tv, j = c
        off = csp.offsets[tv] + 7 * j
        return x[:, off:off + 7]

    def placement_T(vi):
        return pose_xyzyaw(var_value(vi))

    fk_cache = {}

    def fk(c):
        if c not in fk_cache:
            fk_cache[c] = forward_kinematics(rob, conf(c))
        return fk_cache[c]

    r_rob = _t(rob.spheres[:, 3])

    def obj_spheres(o, T):
        s = spec.objects[o].spheres
        return transform_points(T, _t(s[:, :3])), _t(s[:, 3])

    def scene_cost(w, r, scene, skip_objs, obbs):
        tot = sphere_obb_cost(w, r, obbs, eta, smooth)
        for o, pv in scene.items():
            if o in skip_objs:
                continue
            wo, ro = obj_spheres(o, placement_T(pv))
            tot = tot + sphere_sphere_cost(w, r, wo, ro, eta, smooth)
        return tot

    Jc = []
    for t in csp.terms:
        if t.kind == "JL":      # Motion: within joint limits, dist_from_bounds
            Jc.append(dist_from_bounds(conf(t.conf), _t(rob.joint_lo), _t(rob.joint_hi)))
        elif t.kind == "CF":    # CFreeTraj / CFreeHold / CFreeTrajHold
            frames = fk(t.conf)
            w = robot_sphere_centers(rob, frames)
            obbs = [b for i, b in enumerate(spec.obbs) if i not in t.excl_obb]
            j = scene_cost(w, r_rob, t.scene, set(t.excl), obbs)
            if t.held is not None:
                o, gv = t.held
                T_obj = frames[:, 8] @ inverse(G[:, gslot[gv]])
                wo, ro = obj_spheres(o, T_obj)
                j = j + scene_cost(wo, ro, t.scene, {o}, spec.obbs)
            Jc.append(j)
        elif t.kind == "SELF":  # robot self-collision: hinge over the robot's sphere pairs
            w = robot_sphere_centers(rob, fk(t.conf))
            ii = torch.as_tensor([a for a, _ in rob.self_pairs], dtype=torch.long)
            jj = torch.as_tensor([b for _, b in rob.self_pairs], dtype=torch.long)
            d = torch.linalg.vector_norm(w[:, ii] - w[:, jj], dim=-1)
            Jc.append(collision_cost(r_rob[ii] + r_rob[jj] + eta - d, eta, smooth).sum(-1))
        elif t.kind in ("KP", "KR"):   # Kin(q, o, g, p): FK(q) = p . g
            target = placement_T(t.placement) @ G[:, gslot[t.grasp]]
            e_pos, e_rot = pose_error(fk(t.conf)[:, 8], target)
            Jc.append(e_pos if t.kind == "KP" else e_rot)
        elif t.kind == "SS":   # StablePlace support: |z_bottom - z_top|
            s = spec.surfaces[t.surface]
            Jc.append((var_value(t.placement)[:, 2] - s.frame[2]).abs())
        elif t.kind == "SC":   # StablePlace containment: sum over spheres of dist_from_bounds (L6)
            s = spec.surfaces[t.surface]
            w, r = obj_spheres(t.obj, placement_T(t.placement))
            c, sn = math.cos(s.frame[3]), math.sin(s.frame[3])
            dx, dy = w[..., 0] - s.frame[0], w[..., 1] - s.frame[1]
            loc = torch.stack([c * dx + sn * dy, -sn * dx + c * dy], -1)     # Rz(-yaw)(w - s)
            lower = _t(s.lo)[None, :] + r[:, None]
            upper = _t(s.hi)[None, :] - r[:, None]
            Jc.append(dist_from_bounds(loc, lower, upper).sum(-1))
        elif t.kind == "PC":   # ValidPress / ValidStickPress contact (R8): the sphere of the
            # pressing object closest to the button face region, dist_from_bounds on the unshrunk face
            s = spec.surfaces[t.surface]
            w, r = obj_spheres(t.obj, placement_T(t.placement))
            c, sn = math.cos(s.frame[3]), math.sin(s.frame[3])
            dx, dy = w[..., 0] - s.frame[0], w[..., 1] - s.frame[1]
            loc = torch.stack([c * dx + sn * dy, -sn * dx + c * dy], -1)
            e = dist_from_bounds(loc, _t(s.lo), _t(s.hi))                 # [N, m]
            Jc.append(e.min(-1).values)
        elif t.kind == "CP":   # CFreePlace(o, p): support excluded (L3)
            s = spec.surfaces[t.surface]
            w, r = obj_spheres(t.obj, placement_T(t.placement))
            obbs = [b for i, b in enumerate(spec.obbs) if i != s.support_obb]
            Jc.append(scene_cost(w, r, t.scene, {t.obj, s.support_obj}, obbs))
        else:
            raise ValueError(t.kind)
    Jc = torch.stack(Jc, -1) if Jc else torch.zeros(N, 0, dtype=DT)
    lam = _t([spec.lam[t.kind] for t in csp.terms])
    soft = torch.zeros(N, dtype=DT)
    if csp.goal:   # MinimizeObjDist goal cost (Listing 2 obj_dist)
        P = torch.stack([var_value(pv)[:, :3] for pv in csp.goal.values()], 1)
        soft = soft + spec.lam_goal * obj_dist(P)
    for q1, tv, q2 in csp.traj_costs:   # TrajLength(tau) (Listing 1 cost)
        seq = [conf(("var", q1))] + [conf(("knot", tv, j)) for j in range(V[tv].n_knots)] + [conf(("var", q2))]
        for a, b in zip(seq[:-1], seq[1:]):
            soft = soft + spec.lam_traj * torch.linalg.vector_norm(b - a, dim=-1)
    J = (Jc * lam).sum(-1) + soft
    return J, Jc, soft


def cost_and_grad(spec, csp, x_np, grasps_np):
    """J, Jc, soft and dJ/dx per particle (autograd of Eq. 2 summed over particles; particles never couple)."""
    x = torch.tensor(x_np, dtype=DT, requires_grad=True)
    J, Jc, soft = evaluate(spec, csp, x, torch.as_tensor(grasps_np, dtype=DT))
    J.sum().backward()
    return J.detach().numpy(), Jc.detach().numpy(), soft.detach().numpy(), x.grad.numpy()


# ----------------------------------------------------------------------------------------------
# Eq. 4 + Adam (Kingma & Ba cited at P:474) + projection to bounds (L11)
# ----------------------------------------------------------------------------------------------
@dataclasses.dataclass
class State:
    x: np.ndarray
    m: np.ndarray
    v: np.ndarray
    t: int
    invalid: np.ndarray
    grasps: np.ndarray


def new_state(x0, grasps):
    N, D = x0.shape
    return State(x=x0.astype(np.float64).copy(), m=np.zeros((N, D)), v=np.zeros((N, D)), t=0,
                 invalid=np.zeros(N, bool), grasps=grasps.astype(np.float64).copy())


def adam_update(spec, csp, st: State, g):
    """One Adam step (Kingma & Ba Alg. 1) on every particle, then clamp to [lo, hi] (L11).

    Particles whose cost or gradient is non-finite become (sticky) invalid and are not updated (§8(b)).
    """
    st.t += 1
    b1, b2, eps = spec.beta1, spec.beta2, spec.adam_eps
    ok = ~st.invalid
    m = b1 * st.m + (1 - b1) * g
    v = b2 * st.v + (1 - b2) * g * g
    mhat = m / (1 - b1 ** st.t)
    vhat = v / (1 - b2 ** st.t)
    x = st.x - csp.lr * mhat / (np.sqrt(vhat) + eps)
    x = np.minimum(np.maximum(x, csp.lo), csp.hi)
    st.x[ok], st.m[ok], st.v[ok] = x[ok], m[ok], v[ok]


def optimize(spec, csp, st: State, n_steps: int, grad_scale: float):
    """OptimizeParticles (Alg. 1): n_steps of Eq. 4 gradient (scaled by 1/N_global, L10) + Adam."""
    for _ in range(n_steps):
        J, _, _, g = cost_and_grad(spec, csp, st.x, st.grasps)
        bad = ~np.isfinite(J) | ~np.all(np.isfinite(g), axis=1)
        st.invalid |= bad
        adam_update(spec, csp, st, grad_scale * g)
    return st


# ----------------------------------------------------------------------------------------------
# Eq. 3 satisfaction, Eq. 5 counts, best-k
# ----------------------------------------------------------------------------------------------
def check(spec, csp, st: State):
    """Returns (class [N] uint8: 0 satisfying, 1 unsatisfied, 2 invalid; counts [n_hard + 2]; J; soft; Jc)."""
    with torch.no_grad():
        J, Jc, soft = evaluate(spec, csp, torch.as_tensor(st.x, dtype=DT), torch.as_tensor(st.grasps, dtype=DT))
    J, Jc, soft = J.numpy(), Jc.numpy(), soft.numpy()
    eps = np.array([spec.eps[t.kind] for t in csp.terms])
    sat_c = Jc <= eps[None, :]                   # NaN compares False (L21: "<=")
    cls = np.where(sat_c.all(axis=1), 0, 1).astype(np.uint8)
    cls[st.invalid | ~np.isfinite(J)] = 2
    counts = np.zeros(len(csp.terms) + 2, dtype=np.int64)
    counts[:len(csp.terms)] = sat_c.sum(axis=0)
    counts[-2] = int((cls == 0).sum())
    counts[-1] = int((cls == 2).sum())
    return cls, counts, J, soft, Jc


def plan_heuristic(counts, penalty):
    """Eq. 5: H = 1/|con| sum_c h(P, c), h = Lambda_penalty if n_satisfying(c) = 0 else n_satisfying(c)."""
    counts = list(counts)
    if not counts:
        return 0.0
    return sum(penalty if n == 0 else n for n in counts) / len(counts)


def best_k(cls, J, soft, gidx, k):
    """Key (class, cost, global index) ascending; cost = soft plan cost if satisfying else J (L19)."""
    cost = np.where(cls == 0, soft, np.where(cls == 1, J, 0.0))
    order = np.lexsort((np.asarray(gidx), cost, cls))
    sel = order[:k]
    return sel, cls[sel], cost[sel]
