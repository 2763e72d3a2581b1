"""Oracle pins: RNG, geometry, residual primitives (CPU only).

Each test pins an oracle function to something other than itself: the paper's / SPEC's worked
examples (tests/golden/spec_examples.txt), published known-answer vectors, closed forms, an
independent library routine (scipy Rotation) or central finite differences.
"""
import math
import os

import numpy as np
import pytest
import torch
from scipy.spatial.transform import Rotation

from oracle import tamp_oracle as O
from oracle.philox import philox4x32_10, uniforms
from workloads import panda_robot
from workloads.scenes import Robot, OBB

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
DT = torch.float64


def test_philox_known_answers():
    """Random123 KAT vectors (tests/golden/philox4x32_10_kat.txt)."""
    n = 0
    for line in open(os.path.join(GOLDEN, "philox4x32_10_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(t, 16) for t in line.split()]
        out = philox4x32_10(np.array(w[:4], dtype=np.uint64), np.array(w[4:6], dtype=np.uint64))
        assert [int(v) for v in out] == w[6:10]
        n += 1
    assert n == 3


def test_uniforms_range_determinism_and_chi2():
    """u in [0,1), deterministic under the seed, chi^2 uniform over 16 bins at N=4096."""
    g = np.arange(4096)
    u1 = uniforms(1234, g, 7, 3)
    u2 = uniforms(1234, g, 7, 3)
    assert np.array_equal(u1, u2)
    assert u1.min() >= 0.0 and u1.max() < 1.0
    assert not np.array_equal(u1, uniforms(1235, g, 7, 3))
    for col in range(3):
        h, _ = np.histogram(u1[:, col], bins=16, range=(0, 1))
        chi2 = ((h - 256.0) ** 2 / 256.0).sum()
        assert chi2 < 37.7       # p = 0.001 critical value for 15 dof


def _planar_robot(links):
    """All joint axes parallel (alpha = 0): the planar special case of the DH chain."""
    dh = np.zeros((7, 3))
    for i, L in enumerate(links):
        dh[i + 1, 0] = L          # a_{j-1} of joint j+1 = link length i
    return Robot(dh=dh, flange_d=0.0, tcp_yaw=0.0, tcp_d=0.0, joint_lo=-np.ones(7) * 4,
                 joint_hi=np.ones(7) * 4, spheres=np.zeros((0, 4)), sphere_link=np.zeros(0, np.int32))


@pytest.mark.parametrize("q,expect", [
    ([0, 0, 0], (3, 0, 0)),
    ([math.pi / 2, 0, 0], (0, 3, math.pi / 2)),
    ([math.pi / 2, -math.pi / 2, 0], (2, 1, 0)),
])
def test_fk_planar_special_case(q, expect):
    """SPEC examples S:64-66: links [1,1,1] planar arm."""
    rob = _planar_robot([1, 1, 1])
    qq = torch.zeros(1, 7, dtype=DT)
    qq[0, :3] = torch.tensor(q, dtype=DT)
    # tip = origin of the frame after the third link: frame 4 (joint 4 at q=0)
    T = O.forward_kinematics(rob, qq)[0, 8]
    yaw = math.atan2(T[1, 0].item(), T[0, 0].item())
    assert T[0, 3].item() == pytest.approx(expect[0], abs=1e-12)
    assert T[1, 3].item() == pytest.approx(expect[1], abs=1e-12)
    assert yaw == pytest.approx(expect[2], abs=1e-12)
    assert T[2, 3].item() == pytest.approx(0.0, abs=1e-12)


def test_fk_panda_zero_config():
    """Public Franka DH at q = 0: flange at (0.088, 0, 0.926), R = diag(1, -1, -1); TCP 0.1034 below."""
    rob = panda_robot()
    F = O.forward_kinematics(rob, torch.zeros(1, 7, dtype=DT))[0]
    flange = F[7] @ O.trans(0.0, 0.0, rob.flange_d)
    np.testing.assert_allclose(flange[:3, 3].numpy(), [0.088, 0.0, 0.926], atol=1e-12)
    np.testing.assert_allclose(flange[:3, :3].numpy(), np.diag([1.0, -1.0, -1.0]), atol=1e-12)
    np.testing.assert_allclose(F[8][:3, 3].numpy(), [0.088, 0.0, 0.926 - 0.1034], atol=1e-12)


def test_fk_jacobian_column_identity_vs_fd():
    """dp/dq_i = z_i x (p - o_i) (revolute Jacobian) against central finite differences."""
    rob = panda_robot()
    rng = np.random.default_rng(0)
    for _ in range(5):
        q = rng.uniform(rob.joint_lo, rob.joint_hi)
        F = O.forward_kinematics(rob, torch.tensor(q[None], dtype=DT))[0]
        p = F[8][:3, 3].numpy()
        h = 1e-6
        for i in range(7):
            qp, qm = q.copy(), q.copy()
            qp[i] += h
            qm[i] -= h
            pp = O.forward_kinematics(rob, torch.tensor(qp[None], dtype=DT))[0, 8][:3, 3].numpy()
            pm = O.forward_kinematics(rob, torch.tensor(qm[None], dtype=DT))[0, 8][:3, 3].numpy()
            fd = (pp - pm) / (2 * h)
            z = F[i + 1][:3, 2].numpy()
            o = F[i + 1][:3, 3].numpy()
            np.testing.assert_allclose(np.cross(z, p - o), fd, atol=1e-8)


def _unit_box():
    return OBB(center=np.zeros(3), yaw=0.0, half=np.ones(3) * 0.5)


def _sphere_box(c, r, obb, eta=0.0):
    w = torch.tensor(np.array(c, float)[None, None], dtype=DT)
    return O.sphere_obb_cost(w, torch.tensor([r], dtype=DT), [obb], eta).item()


def test_sphere_box_spec_examples():
    """S:82-84."""
    box = _unit_box()
    assert _sphere_box([10, 10, 0], 0.1, box) == 0.0
    assert _sphere_box([0.5, 0.0, 0.0], 0.1, box) == pytest.approx(0.1, abs=1e-15)
    assert _sphere_box([0.55, 0.0, 0.0], 0.1, box) == pytest.approx(0.05, abs=1e-15)


def test_box_signed_distance_closed_forms_and_brute_force():
    """Face region = normal distance; edge = sqrt(dx^2 + dy^2); inside = -(min face distance);
    outside also equals the distance to the clamp-projected closest point (independent formula)."""
    rng = np.random.default_rng(1)
    for _ in range(200):
        yaw = rng.uniform(-math.pi, math.pi)
        half = rng.uniform(0.05, 0.5, 3)
        ctr = rng.normal(0, 0.3, 3)
        obb = OBB(center=ctr, yaw=yaw, half=half)
        c_, R, h = O.obb_arrays(obb)
        Rn = R.numpy()
        pl = rng.uniform(-1.5, 1.5, 3) * half          # local point
        w = Rn @ pl + ctr
        sd = O.box_signed_distance(torch.tensor(w[None]), c_, R, h).item()
        q = np.clip(pl, -half, half)
        if np.any(np.abs(pl) > half):
            assert sd == pytest.approx(np.linalg.norm(pl - q), abs=1e-12)
        else:
            assert sd == pytest.approx(-np.min(half - np.abs(pl)), abs=1e-12)
    # explicit edge region
    box = _unit_box()
    c_, R, h = O.obb_arrays(box)
    sd = O.box_signed_distance(torch.tensor([[0.8, 0.9, 0.0]], dtype=DT), c_, R, h).item()
    assert sd == pytest.approx(math.hypot(0.3, 0.4), abs=1e-15)


def test_sphere_sphere_and_empty_world():
    """S:151 (two r=0.1 spheres at 0.15 -> 0.05), S:150 (empty world -> 0)."""
    wa = torch.tensor([[[0.0, 0.0, 0.0]]], dtype=DT)
    wb = torch.tensor([[[0.15, 0.0, 0.0]]], dtype=DT)
    r = torch.tensor([0.1], dtype=DT)
    assert O.sphere_sphere_cost(wa, r, wb, r, 0.0).item() == pytest.approx(0.05, abs=1e-15)
    assert O.sphere_obb_cost(wa, r, [], 0.0).item() == 0.0


def test_dist_from_bounds_examples():
    """S:91-93 and the Listing 2 semantics."""
    f = lambda v, lo, hi: O.dist_from_bounds(torch.tensor(v, dtype=DT), torch.tensor(lo, dtype=DT),
                                             torch.tensor(hi, dtype=DT)).item()
    assert f([0.5], [0.0], [1.0]) == 0.0
    assert f([4.0, 5.0], [0.0, 0.0], [1.0, 1.0]) == pytest.approx(5.0, abs=1e-15)
    assert f([1.0, 0.0], [0.0, 0.0], [1.0, 1.0]) == 0.0
    assert f([-3.0, 0.5], [0.0, 0.0], [1.0, 1.0]) == pytest.approx(3.0, abs=1e-15)


def test_obj_dist_examples():
    """S:186-188."""
    P0 = torch.zeros(1, 3, 3, dtype=DT)
    assert O.obj_dist(P0).item() == 0.0
    P1 = torch.tensor([[[0.0, 0, 0], [2.0, 0, 0]]], dtype=DT)
    assert O.obj_dist(P1).item() == pytest.approx(2.0, abs=1e-15)
    s3 = math.sqrt(3) / 2
    P2 = torch.tensor([[[0.0, 0, 0], [1.0, 0, 0], [0.5, s3, 0]]], dtype=DT)
    assert O.obj_dist(P2).item() == pytest.approx(3.0, abs=1e-14)


def test_rotation_angle_vs_scipy_and_offsets():
    """Geodesic angle (L4) equals scipy's rotation-vector magnitude of Ra^T Rb; pure offsets."""
    rng = np.random.default_rng(2)
    A = Rotation.random(300, random_state=3)
    B = Rotation.random(300, random_state=4)
    th = O.rotation_angle(torch.tensor(A.as_matrix()), torch.tensor(B.as_matrix())).numpy()
    ref = (A.inv() * B).magnitude()
    np.testing.assert_allclose(th, ref, atol=1e-12)
    for ang in (1e-4, 0.05, 0.1, 1.0, 3.0):
        axis = rng.normal(size=3)
        axis /= np.linalg.norm(axis)
        Ra = Rotation.random(random_state=5).as_matrix()
        Rb = Ra @ Rotation.from_rotvec(ang * axis).as_matrix()
        v = O.rotation_angle(torch.tensor(Ra[None]), torch.tensor(Rb[None])).item()
        assert v == pytest.approx(ang, rel=1e-10)


def test_collision_rigid_transform_invariance():
    """Collision costs are invariant under a rigid motion of all geometry."""
    rng = np.random.default_rng(6)
    w = rng.normal(0, 0.3, (1, 20, 3))
    r = rng.uniform(0.02, 0.1, 20)
    obb = OBB(center=np.array([0.1, -0.2, 0.05]), yaw=0.3, half=np.array([0.2, 0.1, 0.3]))
    base = O.sphere_obb_cost(torch.tensor(w), torch.tensor(r), [obb], 0.0).item()
    ang, t = 0.7, np.array([0.3, -1.0, 0.2])
    Rz = np.array([[math.cos(ang), -math.sin(ang), 0], [math.sin(ang), math.cos(ang), 0], [0, 0, 1]])
    w2 = w @ Rz.T + t
    obb2 = OBB(center=Rz @ obb.center + t, yaw=obb.yaw + ang, half=obb.half)
    moved = O.sphere_obb_cost(torch.tensor(w2), torch.tensor(r), [obb2], 0.0).item()
    assert base > 0
    assert moved == pytest.approx(base, rel=1e-12)
    wb = rng.normal(0, 0.3, (1, 7, 3))
    rb = rng.uniform(0.02, 0.1, 7)
    s1 = O.sphere_sphere_cost(torch.tensor(w), torch.tensor(r), torch.tensor(wb), torch.tensor(rb), 0.0).item()
    s2 = O.sphere_sphere_cost(torch.tensor(w2), torch.tensor(r), torch.tensor(wb @ Rz.T + t), torch.tensor(rb), 0.0).item()
    assert s1 == pytest.approx(s2, rel=1e-12)


def test_top_down_grasp_frame():
    """T(g) = Trans Rz(gamma) Rx(pi): orthonormal, approach axis (z) points down (top-down)."""
    T = O.top_down_grasp(torch.tensor([0.01], dtype=DT), torch.tensor([-0.02], dtype=DT),
                         torch.tensor([0.03], dtype=DT), torch.tensor([0.4], dtype=DT))[0].numpy()
    R = T[:3, :3]
    np.testing.assert_allclose(R @ R.T, np.eye(3), atol=1e-14)
    np.testing.assert_allclose(R[:, 2], [0, 0, -1], atol=1e-14)
    np.testing.assert_allclose(T[:3, 3], [0.01, -0.02, 0.03], atol=1e-15)
    assert math.atan2(R[1, 0], R[0, 0]) == pytest.approx(0.4, abs=1e-14)


def _rx(a):
    c, s = math.cos(a), math.sin(a)
    return np.array([[1, 0, 0], [0, c, -s], [0, s, c]], float)


def test_full_orientation_box_closed_forms():
    """Oriented boxes with a full rotation.  (a) A box turned by Rx(pi/2) with half extents (a, b, c)
    occupies the same points as the axis-aligned box with half extents (a, c, b): the sphere cost of any sphere is
    the same.  (b) A unit cube turned 45 degrees about x: a sphere straight above the centre at height z sees the
    top edge at sqrt(2)/2, so its hinge is r - (z - sqrt(2)/2).  (c) The full-rotation form with R = Rz(yaw) equals
    the yaw form."""
    rng = np.random.default_rng(3)
    half = np.array([0.3, 0.1, 0.2])
    tilted = OBB(center=np.array([0.1, 0.2, 0.3]), yaw=0.0, half=half, R=_rx(math.pi / 2))
    flat = OBB(center=np.array([0.1, 0.2, 0.3]), yaw=0.0, half=half[[0, 2, 1]])
    w = torch.tensor(rng.uniform(-0.6, 0.8, (1, 200, 3)))
    r = torch.tensor(rng.uniform(0.02, 0.15, 200))
    a = O.sphere_obb_cost(w, r, [tilted], 0.0).item()
    b_ = O.sphere_obb_cost(w, r, [flat], 0.0).item()
    assert a > 0.1 and a == pytest.approx(b_, rel=1e-12)
    cube = OBB(center=np.zeros(3), yaw=0.0, half=np.full(3, 0.5), R=_rx(math.pi / 4))
    for z, rad in ((0.8, 0.2), (1.0, 0.4), (0.75, 0.1)):
        v = _sphere_box([0.0, 0.0, z], rad, cube)
        assert v == pytest.approx(max(0.0, rad - (z - math.sqrt(0.5))), abs=1e-12)
    yawed = OBB(center=np.array([0.2, -0.1, 0.0]), yaw=0.6, half=half)
    c, s = math.cos(0.6), math.sin(0.6)
    full = OBB(center=yawed.center, yaw=0.0, half=half, R=np.array([[c, -s, 0], [s, c, 0], [0, 0, 1.0]]))
    assert O.sphere_obb_cost(w, r, [yawed], 0.0).item() == pytest.approx(O.sphere_obb_cost(w, r, [full], 0.0).item(),
                                                                           rel=1e-12)


def test_full_orientation_rigid_invariance():
    """Sphere-box costs are invariant under a rigid motion of the spheres and a fully rotated box."""
    rng = np.random.default_rng(7)
    w = rng.normal(0, 0.3, (1, 30, 3))
    r = rng.uniform(0.02, 0.1, 30)
    R0 = Rotation.random(random_state=8).as_matrix()
    box = OBB(center=np.array([0.05, -0.1, 0.1]), yaw=0.0, half=np.array([0.25, 0.1, 0.3]), R=R0)
    base = O.sphere_obb_cost(torch.tensor(w), torch.tensor(r), [box], 0.0).item()
    Q = Rotation.random(random_state=9).as_matrix()
    t = np.array([0.3, -1.0, 0.2])
    box2 = OBB(center=Q @ box.center + t, yaw=0.0, half=box.half, R=Q @ R0)
    moved = O.sphere_obb_cost(torch.tensor(w @ Q.T + t), torch.tensor(r), [box2], 0.0).item()
    assert base > 0 and moved == pytest.approx(base, rel=1e-12)
