"""Closed-form pins of the oracle's term assembly (CPU only).

Each test fixes one part of `oracle/tamp_oracle.py` against a value worked out by hand from the paper's
definition for a hand-placed configuration -- not by re-calling the oracle's own formula:

* StablePlace containment SC ("contained", Listing 2 `dist_from_bounds` P:1592-1606, reading L6):
  a block straddling the region's corner by a known excess per sphere, in a yawed surface frame;
* CFreePlace CP ignores its support only (reading L3): a block sunk 1 mm into its support
  table / support object and pushed 2 mm into a wall;
* TrajLength (Listing 1 cost): straight-line knots sum to ||q2 - q1||, a displaced middle
  knot to the closed form;
* the weighted goal cost lambda_goal * obj_dist (Listing 2; S:188's unit
  equilateral triangle gives 3, so 3 lambda_goal; a square of side s gives s (4 + 2 sqrt 2));
* the held object at a MoveHold knot at T_ee T(g)^-1 (CFreeTrajHold): a box under the lowest held
  sphere at a known depth, sphere positions composed by hand with numpy's matrix inverse;
* robot collision spheres on their link frames: world centres at q = 0 against the frames of
  the public modified-DH table worked out by hand (and rotated by pi/2 about the base axis).
"""
import copy
import math

import numpy as np
import pytest
import torch

from oracle import tamp_oracle as O
from workloads import make_config
from workloads.scenes import OBB, Surface, PLACEMENT, CONF, TRAJ, MOVE_FREE, MOVE_HOLD

DT = torch.float64


def _eval(spec, csp, x, g):
    with torch.no_grad():
        J, Jc, soft = O.evaluate(spec, csp, torch.as_tensor(x, dtype=DT), torch.as_tensor(g, dtype=DT))
    return J.numpy(), Jc.numpy(), soft.numpy()


def _term(csp, kind, k=0):
    return [i for i, t in enumerate(csp.terms) if t.kind == kind][k]


def _identity_grasps(csp, n=1):
    g = np.zeros((n, len(csp.grasp_vars), 3, 4))
    g[..., 0, 0] = g[..., 1, 1] = g[..., 2, 2] = 1.0
    return g


# ---------------------------------------------------------------------------------------------------
# StablePlace containment (SC)
# ---------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("psi", [0.0, 0.3, -2.2])
def test_sc_block_straddling_region_corner(psi):
    """Config 1's 5 cm block (8 spheres of r = 1.25 cm at (+-1.25, +-1.25) cm) placed with its centre at local
    (0.0875 + e, 0.0875 + e) (and its mirror image) in a 20x20 cm region (lo = -0.1, hi = 0.1) whose frame is yawed by psi, the block
    aligned with the frame.  Shrunk bound hi - r = 0.0875, so the +x spheres stick out by 0.0125 + e in x,
    the +y spheres by 0.0125 + e in y, the -x / -y ones not at all:
        SC = 2 levels x ((0.0125 + e) sqrt 2 + 2 (0.0125 + e))."""
    spec = make_config(1, n=1)
    e = 0.004
    frame = np.array([0.5, 0.2, 0.0, psi])
    spec.surfaces = [Surface("region", frame, np.array([-0.1, -0.1]), np.array([0.1, 0.1]), support_obb=0)]
    csp = O.build_csp(spec)
    i_sc = _term(csp, "SC")
    vp = csp.terms[i_sc].placement
    lx = ly = 0.0875 + e
    c, s = math.cos(psi), math.sin(psi)
    x = np.zeros((1, csp.D))
    x[0, csp.offsets[vp]:csp.offsets[vp] + 4] = [0.5 + c * lx - s * ly, 0.2 + s * lx + c * ly, 0.0, psi]
    _, Jc, _ = _eval(spec, csp, x, _identity_grasps(csp))
    ex = 0.0125 + e
    assert Jc[0, i_sc] == pytest.approx(2 * (ex * math.sqrt(2) + 2 * ex), abs=1e-8)
    # the mirrored corner (lo side: lo + r = -0.0875)
    x[0, csp.offsets[vp]:csp.offsets[vp] + 2] = [0.5 - c * lx + s * ly, 0.2 - s * lx - c * ly]
    assert _eval(spec, csp, x, _identity_grasps(csp))[1][0, i_sc] == \
        pytest.approx(2 * (ex * math.sqrt(2) + 2 * ex), abs=1e-8)
    # fully inside the shrunk region -> exactly 0; +x sphere centres on the (unshrunk) edge -> r each
    x[0, csp.offsets[vp]:csp.offsets[vp] + 2] = [0.5, 0.2]
    assert _eval(spec, csp, x, _identity_grasps(csp))[1][0, i_sc] == 0.0
    lx, ly = 0.0875, 0.0                   # +x sphere centres on the region edge: excess r each
    x[0, csp.offsets[vp]:csp.offsets[vp] + 2] = [0.5 + c * lx - s * ly, 0.2 + s * lx + c * ly]
    assert _eval(spec, csp, x, _identity_grasps(csp))[1][0, i_sc] == pytest.approx(4 * 0.0125, abs=1e-8)


# ---------------------------------------------------------------------------------------------------
# CFreePlace (CP): support excluded, everything else counted
# ---------------------------------------------------------------------------------------------------
def test_cp_ignores_support_table_but_not_a_wall():
    """Config 1's block placed 1 mm *into* its support table (z = -0.001): its 4 bottom spheres (centres
    1.15 cm above the table top, r = 1.25 cm) would penetrate the table by 1 mm each, but the support is
    excluded (L3), so CP = 0.  A wall (not the support) whose face is 2 mm inside the block's +x face adds
    4 spheres x 2 mm = 0.008 exactly."""
    spec = make_config(1, n=1)
    csp = O.build_csp(spec)
    i_cp = _term(csp, "CP")
    vp = csp.terms[i_cp].placement
    sf = spec.surfaces[csp.terms[i_cp].surface]
    assert sf.support_obb == 0
    px, py = sf.frame[0], sf.frame[1]
    x = np.zeros((1, csp.D))
    x[0, csp.offsets[vp]:csp.offsets[vp] + 4] = [px, py, -0.001, 0.0]
    g = _identity_grasps(csp)
    assert _eval(spec, csp, x, g)[1][0, i_cp] == 0.0
    wall = OBB(center=np.array([px + 0.025 - 0.002 + 0.005, py, 0.05]), yaw=0.0,
               half=np.array([0.005, 0.2, 0.05]), name="wall")
    spec.obbs = spec.obbs + [wall]
    assert _eval(spec, csp, x, g)[1][0, i_cp] == pytest.approx(4 * 0.002, abs=1e-8)


def test_cp_ignores_support_object_but_not_other_objects():
    """Config 2's red block stacked on blue and sunk 5 mm into it: red's bottom spheres (r = 1.25 cm at
    (+-1.25, +-1.25, 8.75) cm) reach blue's top spheres (r = 2 cm at (+-2, +-2, 6) cm): distance
    sqrt(2 * 0.0075^2 + 0.0275^2) < 0.0325, but blue is the support (L3), so CP = 0 with the obstructors
    parked far away.  Parking obstructor A on top of red makes CP positive."""
    spec = make_config(2, n=1)
    csp = O.build_csp(spec)
    i_cp = _term(csp, "CP", 2)                     # red onto blue
    t = csp.terms[i_cp]
    sf = spec.surfaces[t.surface]
    assert sf.support_obj == 0 and t.obj == 3
    x = np.zeros((1, csp.D))
    bx, by = sf.frame[0], sf.frame[1]
    x[0, csp.offsets[t.placement]:csp.offsets[t.placement] + 4] = [bx, by, 0.08 - 0.005, 0.0]
    pa, pb = [vi for vi, v in enumerate(spec.variables) if v.kind == PLACEMENT and not v.const][:2]
    x[0, csp.offsets[pa]:csp.offsets[pa] + 4] = [0.2, 0.6, 0.0, 0.0]
    x[0, csp.offsets[pb]:csp.offsets[pb] + 4] = [0.5, 0.6, 0.0, 0.0]
    g = _identity_grasps(csp)
    d = math.sqrt(2 * 0.0075 ** 2 + 0.0275 ** 2)
    assert 0.0325 - d > 1e-3                        # would penetrate if blue were not excluded
    assert _eval(spec, csp, x, g)[1][0, i_cp] == 0.0
    # obstructor A's bottom spheres (r = 1.25 cm at (+-1.25, +-1.25, 1.25) cm) 2 cm above red's top spheres
    # (z = 0.075 + 0.0375): vertical distance 0.02 < 0.025 -> 4 pairs of 5 mm each (the other pairs are
    # >= sqrt(0.025^2 + 0.02^2) = 0.032 apart)
    x[0, csp.offsets[pa]:csp.offsets[pa] + 4] = [bx, by, 0.075 + 0.0375 + 0.02 - 0.0125, 0.0]
    assert _eval(spec, csp, x, g)[1][0, i_cp] == pytest.approx(4 * 0.005, abs=1e-8)


# ---------------------------------------------------------------------------------------------------
# TrajLength
# ---------------------------------------------------------------------------------------------------
def _motions(spec):
    return [a for a in spec.actions if a.kind in (MOVE_FREE, MOVE_HOLD) and a.traj >= 0
            and spec.variables[a.traj].n_knots > 0]


def test_traj_length_straight_and_bent_knots():
    """Config 4 (every motion carries 3 free knots, no goal cost): with the knots on the straight line
    from q1 to q2 each motion contributes lambda_traj ||q2 - q1|| (q1 = the constant q0 for the first
    motion); moving one motion's middle knot by d orthogonal to delta = q2 - q1 changes its length to
    ||delta||/2 + 2 sqrt(||delta||^2/16 + ||d||^2)."""
    spec = make_config(4, n=1)
    assert not spec.goal_objs
    csp = O.build_csp(spec)
    rng = np.random.default_rng(3)
    x = rng.uniform(-1.0, 1.0, (1, csp.D))
    V = spec.variables

    def qval(vi):
        return np.asarray(V[vi].value, float) if V[vi].const else x[0, csp.offsets[vi]:csp.offsets[vi] + 7]

    mot = _motions(spec)
    assert len(mot) == 12
    total = 0.0
    for a in mot:
        q1, q2 = qval(a.q1), qval(a.q2)
        K = V[a.traj].n_knots
        for j in range(K):
            x[0, csp.offsets[a.traj] + 7 * j:csp.offsets[a.traj] + 7 * j + 7] = q1 + (j + 1) / (K + 1) * (q2 - q1)
        total += np.linalg.norm(q2 - q1)
    g = np.tile(_identity_grasps(csp), 1)
    soft = _eval(spec, csp, x, g)[2][0]
    assert soft == pytest.approx(spec.lam_traj * total, rel=1e-12)
    # bend the middle knot of the third motion
    a = mot[2]
    q1, q2 = qval(a.q1), qval(a.q2)
    delta = q2 - q1
    d = rng.normal(size=7)
    d -= d @ delta / (delta @ delta) * delta
    d *= 0.3 / np.linalg.norm(d)
    off = csp.offsets[a.traj] + 7
    x[0, off:off + 7] += d
    L = np.linalg.norm(delta)
    bent = total - L + L / 2 + 2 * math.sqrt(L * L / 16 + 0.09)
    assert _eval(spec, csp, x, g)[2][0] == pytest.approx(spec.lam_traj * bent, rel=1e-12)


# ---------------------------------------------------------------------------------------------------
# weighted goal cost (MinimizeObjDist)
# ---------------------------------------------------------------------------------------------------
def test_goal_cost_weighted_obj_dist():
    """Config 3's goal cost lambda_goal * obj_dist (reading L7: lambda_goal = 0.025).  Final
    placements of four goal objects at the corners of a 10 cm square: obj_dist = 0.1 (4 + 2 sqrt 2) (four sides, two
    diagonals; L24 uses xyz, so equal z); three on a unit equilateral triangle: obj_dist = 3, soft = 3 lambda.
    J = sum lambda_c J_c + soft (Eq. 2)."""
    spec = make_config(3, n=1)
    lam = spec.lam_goal
    assert lam == pytest.approx(0.025, rel=1e-7)
    csp = O.build_csp(spec)
    goal_vars = list(csp.goal.values())
    assert len(goal_vars) == 4
    x = np.zeros((1, csp.D))
    sq = [(0.0, 0.0), (0.1, 0.0), (0.1, 0.1), (0.0, 0.1)]
    for (px, py), vi in zip(sq, goal_vars):
        x[0, csp.offsets[vi]:csp.offsets[vi] + 4] = [0.4 + px, 0.2 + py, 0.0, 0.7]
    g = _identity_grasps(csp)
    J, Jc, soft = _eval(spec, csp, x, g)
    assert soft[0] == pytest.approx(lam * 0.1 * (4 + 2 * math.sqrt(2)), rel=1e-12)
    lamc = np.array([spec.lam[t.kind] for t in csp.terms])
    assert J[0] == pytest.approx((lamc * Jc[0]).sum() + soft[0], rel=1e-12)
    # three goal objects on a unit equilateral triangle
    spec3 = copy.deepcopy(spec)
    spec3.goal_objs = spec.goal_objs[:3]
    csp3 = O.build_csp(spec3)
    tri = [(0.0, 0.0), (1.0, 0.0), (0.5, math.sqrt(3) / 2)]
    for (px, py), vi in zip(tri, list(csp3.goal.values())):
        x[0, csp3.offsets[vi]:csp3.offsets[vi] + 4] = [px, py, 0.0, 0.0]
    assert _eval(spec3, csp3, x, g)[2][0] == pytest.approx(3 * lam, rel=1e-12)


# ---------------------------------------------------------------------------------------------------
# held object at a MoveHold knot: T_ee T(g)^-1
# ---------------------------------------------------------------------------------------------------
def _rand_rot(rng):
    a = rng.normal(size=(3, 3))
    Q, R = np.linalg.qr(a)
    Q = Q @ np.diag(np.sign(np.diag(R)))
    if np.linalg.det(Q) < 0:
        Q[:, 0] = -Q[:, 0]
    return Q


def test_held_object_at_knot_is_attached_by_inverse_grasp():
    """Config 4's first MoveHold knot with the robot's spheres shrunk to radius 0 and the scene emptied:
    the CF term then sees only the held object.  Its spheres are at T_ee T(g)^-1 c, composed here
    with numpy's 4x4 matrix inverse from the tool frame and a random 6-DOF grasp.  A 40x40 cm box whose top
    face is 1 mm above the bottom of the lowest held sphere makes CF = 1 mm exactly (all other held
    spheres clear by more than 1 mm, every robot sphere centre above the box)."""
    spec = make_config(4, n=1)
    rob = spec.robot
    rob.spheres = rob.spheres.copy()
    rob.spheres[:, 3] = 0.0
    spec.obbs = []
    csp = O.build_csp(spec)
    k = [i for i, t in enumerate(csp.terms) if t.kind == "CF" and t.held is not None][0]
    term = csp.terms[k]
    term.scene = {}
    obj, gv = term.held
    gslot = csp.grasp_vars.index(gv)
    sph = spec.objects[obj].spheres
    rng = np.random.default_rng(5)
    for _ in range(200):
        q = rng.uniform(rob.joint_lo, rob.joint_hi)
        Tg = np.eye(4)
        Tg[:3, :3] = _rand_rot(rng)
        Tg[:3, 3] = rng.uniform(-0.03, 0.03, 3)
        F = O.forward_kinematics(rob, torch.tensor(q[None]))[0].numpy()
        T_obj = F[8] @ np.linalg.inv(Tg)
        w = (T_obj[:3, :3] @ sph[:, :3].T).T + T_obj[:3, 3]
        bottoms = w[:, 2] - sph[:, 3]
        order = np.argsort(bottoms)
        lo_i = order[0]
        rw = O.robot_sphere_centers(rob, torch.tensor(F[None]))[0].numpy()
        ztop = bottoms[lo_i] + 1e-3
        cx, cy = w[lo_i, 0], w[lo_i, 1]
        inside = (np.abs(rw[:, 0] - cx) < 0.2) & (np.abs(rw[:, 1] - cy) < 0.2)
        near = (np.abs(w[:, 0] - cx) < 0.2 - 0.02) & (np.abs(w[:, 1] - cy) < 0.2 - 0.02)
        if (bottoms[order[1]] - bottoms[lo_i] > 2e-3 and np.all(rw[inside, 2] > ztop + 1e-3)
                and np.all(near) and ztop > 0.05):
            break
    else:
        pytest.fail("no admissible random configuration")
    spec.obbs = [OBB(center=np.array([cx, cy, ztop - 0.05]), yaw=0.0, half=np.array([0.2, 0.2, 0.05]))]
    vi, j = term.conf[1], term.conf[2]
    x = np.zeros((1, csp.D))
    x[0, csp.offsets[vi] + 7 * j:csp.offsets[vi] + 7 * j + 7] = q
    g = _identity_grasps(csp)
    g[0, gslot] = Tg[:3]
    _, Jc, _ = _eval(spec, csp, x, g)
    assert Jc[0, k] == pytest.approx(1e-3, abs=1e-8)


# ---------------------------------------------------------------------------------------------------
# robot spheres on their link frames
# ---------------------------------------------------------------------------------------------------
def _panda_frames_q0():
    """Link frames 1..7 and the tool frame of the public modified-DH Panda at q = 0, worked out by hand:
    frame j = frame j-1 . Rx(alpha_j) Tx(a_j) Tz(d_j):  R1 = I, R2 = Rx(-pi/2), R3 = I, R4 = Rx(pi/2), R5 = I,
    R6 = Rx(pi/2), R7 = Rx(pi); origins (0,0,.333) x2, (0,0,.649), (.0825,0,.649), (0,0,1.033) x2,
    (.088,0,1.033); tool = R7 Rz(-pi/4) at 0.107 + 0.1034 below frame 7's origin."""
    I = np.eye(3)
    rxm = np.array([[1, 0, 0], [0, 0, 1], [0, -1, 0]], float)      # Rx(-pi/2)
    rxp = np.array([[1, 0, 0], [0, 0, -1], [0, 1, 0]], float)      # Rx(pi/2)
    rxpi = np.diag([1.0, -1.0, -1.0])
    h = math.sqrt(0.5)
    tool_R = np.array([[h, h, 0], [h, -h, 0], [0, 0, -1]])           # Rx(pi) Rz(-pi/4)
    Rs = [None, I, rxm, I, rxp, I, rxp, rxpi, tool_R]
    ts = [None, (0, 0, .333), (0, 0, .333), (0, 0, .649), (.0825, 0, .649), (0, 0, 1.033), (0, 0, 1.033),
          (.088, 0, 1.033), (.088, 0, 1.033 - 0.107 - 0.1034)]
    return Rs, [None if t is None else np.array(t, float) for t in ts]


@pytest.mark.parametrize("yaw", [0.0, math.pi / 2])
def test_robot_sphere_centres_on_their_link_frames(yaw):
    """w_s = R_link(s) c_s + t_link(s) at q = (yaw, 0, ..., 0): joint 1's axis is the world z axis
    through the base, so every frame is the q = 0 frame rotated by Rz(yaw)."""
    rob = make_config(1, n=1).robot
    q = np.zeros((1, 7))
    q[0, 0] = yaw
    W = O.robot_sphere_centers(rob, O.forward_kinematics(rob, torch.tensor(q))).numpy()[0]
    Rs, ts = _panda_frames_q0()
    c, s = math.cos(yaw), math.sin(yaw)
    Rz = np.array([[c, -s, 0], [s, c, 0], [0, 0, 1.0]])
    assert len(W) == 32 and set(rob.sphere_link.tolist()) == set(range(1, 9))
    for k in range(len(W)):
        link = int(rob.sphere_link[k])
        exp = Rz @ (Rs[link] @ rob.spheres[k, :3] + ts[link])
        np.testing.assert_allclose(W[k], exp, atol=1e-6)
