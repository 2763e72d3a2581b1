"""Oracle pins: skeleton -> CSP, Eq. 2/3/4, Adam, samplers, best-k (CPU only)."""
import copy
import dataclasses
import math

import numpy as np
import pytest
import torch

from oracle import tamp_oracle as O
from workloads import make_config
from workloads.scenes import Surface, PLACEMENT, CONF, PRESS, PRESS_STICK

DT = torch.float64


def _eval(spec, csp, x, g):
    with torch.no_grad():
        J, Jc, soft = O.evaluate(spec, csp, torch.as_tensor(x, dtype=DT), torch.as_tensor(g, dtype=DT))
    return J.numpy(), Jc.numpy(), soft.numpy()


# ---------------------------------------------------------------------------------------------
# skeleton -> constraint network
# ---------------------------------------------------------------------------------------------
def test_running_example_constraint_set():
    """Running example: 10 constraints over free vars q1, tau1, g, q2, tau2, p1.
    Deferred motion drops tau; Grasp(red, g) is identically 0 for sampled grasps.
    The oracle's hard terms: Motion->JL, CFreeTraj+CFreeHold->CF, Kin->KP+KR per conf, StablePlace->SS+SC,
    CFreePlace->CP: 11 terms (SURVEY §8(c) term table)."""
    spec = make_config(1, n=4)
    csp = O.build_csp(spec)
    kinds = [t.kind for t in csp.terms]
    assert kinds == ["JL", "CF", "KP", "KR", "JL", "CF", "KP", "KR", "SS", "SC", "CP"]
    assert csp.D == 7 + 7 + 4
    assert len(csp.grasp_vars) == 1
    # both robot checks exclude the manipulated object (L3)
    assert csp.terms[1].excl == (0,) and csp.terms[5].excl == (0,)
    # the pick's Kin targets the constant initial placement p0, the place's the variable p1
    assert spec.variables[csp.terms[2].placement].const
    assert not spec.variables[csp.terms[6].placement].const


@pytest.mark.parametrize("cfg,D,n_hard,n_grasp", [(1, 18, 11, 1), (2, 54, 33, 3), (3, 72, 44, 4),
                                                  (4, 360, 138, 6), (5, 72, 44, 4), (6, 29, 17, 2),
                                                  (7, 22, 12, 1)])
def test_config_sizes(cfg, D, n_hard, n_grasp):
    """D, hard terms (config 4: 66 + 72 knot terms), frozen grasps."""
    spec = make_config(cfg, n=4)
    csp = O.build_csp(spec)
    assert (csp.D, len(csp.terms), len(csp.grasp_vars)) == (D, n_hard, n_grasp)


# ---------------------------------------------------------------------------------------------
# hand-constructed satisfying particle (SURVEY §8(c) "Whole step" pin)
# ---------------------------------------------------------------------------------------------
def _clear_pickplace():
    """Config 1 in an empty world (no OBBs), large goal region on z = 0."""
    spec = make_config(1, n=4)
    spec.obbs = []
    spec.surfaces = [Surface("big", np.array([0.0, 0.0, 0.0, 0.0]), np.array([-2.0, -2.0]),
                             np.array([2.0, 2.0]))]
    for a in spec.actions:
        if a.surface >= 0:
            a.surface = 0
    for v in spec.variables:
        if v.kind == PLACEMENT and not v.const:
            v.surface = 0
    return spec


def satisfying_particle(spec, csp, rng, psi=0.6):
    """q_pick random; T(g) := T(p0)^-1 FK(q_pick); place = everything rotated by psi about the
    base axis: p1 = Rz(psi) p0, q_place = q_pick + psi e_1 (joint 1 is the world z axis through the base)."""
    rob = spec.robot
    lo, hi = rob.joint_lo.copy(), rob.joint_hi.copy()
    lo[0] += 0.7
    hi[0] -= 0.7
    q = rng.uniform(lo, hi)
    p0 = spec.variables[csp.terms[2].placement].value
    T0 = O.pose_xyzyaw(torch.tensor(p0))
    F = O.forward_kinematics(rob, torch.tensor(q[None]))[0, 8]
    Tg = (O.inverse(T0) @ F).numpy()[:3]
    c, s = math.cos(psi), math.sin(psi)
    p1 = np.array([c * p0[0] - s * p0[1], s * p0[0] + c * p0[1], p0[2], p0[3] + psi])
    x = np.zeros(csp.D)
    vq1, vq2, vp = csp.terms[0].conf[1], csp.terms[4].conf[1], csp.terms[8].placement
    x[csp.offsets[vq1]:csp.offsets[vq1] + 7] = q
    q2 = q.copy()
    q2[0] += psi
    x[csp.offsets[vq2]:csp.offsets[vq2] + 7] = q2
    x[csp.offsets[vp]:csp.offsets[vp] + 4] = p1
    return x, Tg


def test_constructed_satisfying_particle():
    spec = _clear_pickplace()
    csp = O.build_csp(spec)
    rng = np.random.default_rng(7)
    xs, gs = [], []
    for _ in range(8):
        x, Tg = satisfying_particle(spec, csp, rng)
        xs.append(x)
        gs.append(Tg[None])
    x, g = np.array(xs), np.array(gs)
    J, Jc, soft = _eval(spec, csp, x, g)
    assert np.all(Jc[:, [0, 1, 4, 5, 8, 9, 10]] == 0.0)      # hinge / bounds terms exactly 0
    assert np.all(Jc <= 1e-9)                               # kin residuals: rounding only
    assert np.all(J <= 1e-8)
    st = O.new_state(x, g)
    cls, counts, *_ = O.check(spec, csp, st)
    assert np.all(cls == 0)
    assert counts[-2] == 8 and np.all(counts[:-2] == 8)


def test_kin_offsets_and_eq2_examples():
    """Translate p1 by 1 cm -> KP = 0.01 with KR = 0 (pure offset); add 0.1 rad to p1's yaw -> KR = 0.1
    exactly (R_ee^T R* = R_g^T Rz(0.1) R_g), contributing lambda_KR * 0.1 = 0.5 to Eq. 2."""
    spec = _clear_pickplace()
    csp = O.build_csp(spec)
    x, Tg = satisfying_particle(spec, csp, np.random.default_rng(8))
    off = csp.offsets[csp.terms[8].placement]
    xt = x.copy()
    xt[off] += 0.01
    _, Jc, _ = _eval(spec, csp, xt[None], Tg[None, None])
    assert Jc[0, 6] == pytest.approx(0.01, abs=1e-9)
    assert Jc[0, 7] == pytest.approx(0.0, abs=1e-9)
    xr = x.copy()
    xr[off + 3] += 0.1
    J, Jc, soft = _eval(spec, csp, xr[None], Tg[None, None])
    assert Jc[0, 7] == pytest.approx(0.1, abs=1e-9)
    assert spec.lam["KR"] * Jc[0, 7] == pytest.approx(0.5, abs=5e-9)
    assert J[0] == pytest.approx(0.5 + spec.lam["KP"] * Jc[0, 6], abs=5e-9)


def test_eq3_boundary_semantics_and_weight_scaling():
    """J_c <= eps is satisfying (L21): support error exactly 1 cm passes, 1 cm + 1e-9 fails;
    doubling every weight doubles J and leaves the mask unchanged."""
    spec = _clear_pickplace()
    csp = O.build_csp(spec)
    x, Tg = satisfying_particle(spec, csp, np.random.default_rng(10))
    st = O.new_state(x[None], Tg[None, None])
    e_ss = spec.eps["SS"]                         # 1 cm (as float32, like every spec constant)
    spec.surfaces[0].frame[2] = -e_ss             # |z_bottom - z_top| = |0 - (-eps)| = eps_SS exactly
    cls, counts, J, soft, Jc = O.check(spec, csp, st)
    assert Jc[0, 8] == e_ss and abs(e_ss - 0.01) < 1e-9
    assert cls[0] == 0 and counts[8] == 1
    spec_b = copy.deepcopy(spec)
    spec_b.surfaces[0].frame[2] = -e_ss - 1e-9
    cls_b, counts_b, *_ = O.check(spec_b, csp, st)
    assert cls_b[0] == 1 and counts_b[8] == 0
    spec2 = copy.deepcopy(spec)
    spec2.lam = {k: 2 * v for k, v in spec.lam.items()}
    cls2, _, J2, _, _ = O.check(spec2, csp, st)
    assert np.array_equal(cls, cls2)
    np.testing.assert_allclose(J2, 2 * J, rtol=1e-14)


def test_collision_exclusions_brute_force():
    """CF at a pick conf excludes the picked object but includes all others at their current poses (L3);
    CP excludes the support surface/object.  Checked against a brute-force per-pair loop."""
    spec = make_config(2, n=2)
    csp = O.build_csp(spec)
    x, g = O.initialize_particles(spec, csp, 5, np.arange(2))
    t_cf = csp.terms[1]                               # CF(q_pick_obsA)
    assert t_cf.kind == "CF" and t_cf.excl == (1,)
    # put obsB exactly onto the robot's TCP at that conf
    q = x[0, csp.offsets[t_cf.conf[1]]:csp.offsets[t_cf.conf[1]] + 7]
    F = O.forward_kinematics(spec.robot, torch.tensor(q[None]))[0]
    tcp = O.robot_sphere_centers(spec.robot, F[None])[0, 28].numpy()     # a hand sphere
    base = _eval(spec, csp, x, g)[1][0, 1]
    spec_b = copy.deepcopy(spec)
    spec_b.objects[2].init_pose = np.array([tcp[0], tcp[1], tcp[2] - 0.05, 0.0])
    spec_b.variables[[i for i, v in enumerate(spec.variables) if v.name == "p0_obsB"][0]].value = \
        spec_b.objects[2].init_pose.copy()
    with_b = _eval(spec_b, csp, x, g)[1][0, 1]
    # brute force: robot spheres vs obsB spheres
    W = O.robot_sphere_centers(spec.robot, F[None])[0].numpy()
    r = spec.robot.spheres[:, 3]
    ob = spec_b.objects[2]
    c, s = math.cos(ob.init_pose[3]), math.sin(ob.init_pose[3])
    add = 0.0
    for i in range(len(W)):
        for sp in ob.spheres:
            wb = np.array([ob.init_pose[0] + c * sp[0] - s * sp[1], ob.init_pose[1] + s * sp[0] + c * sp[1],
                           ob.init_pose[2] + sp[2]])
            add += max(0.0, r[i] + sp[3] - np.linalg.norm(W[i] - wb))
    old_b = 0.0
    ob0 = spec.objects[2]
    for i in range(len(W)):
        for sp in ob0.spheres:
            wb = ob0.init_pose[:3] + np.array([sp[0], sp[1], sp[2]])
            old_b += max(0.0, r[i] + sp[3] - np.linalg.norm(W[i] - wb))
    assert add > 1e-3
    assert with_b == pytest.approx(base - old_b + add, rel=1e-10, abs=1e-12)
    # moving the excluded (picked) object onto the robot changes nothing
    spec_a = copy.deepcopy(spec)
    spec_a.variables[[i for i, v in enumerate(spec.variables) if v.name == "p0_obsA"][0]].value = \
        np.array([tcp[0], tcp[1], tcp[2] - 0.05, 0.0])
    assert _eval(spec_a, csp, x, g)[1][0, 1] == base
    # CP of red on blue excludes blue (support object) and the table is not the support there
    t_cp = csp.terms[-1]
    assert t_cp.kind == "CP" and spec.surfaces[t_cp.surface].support_obj == 0


def test_permutation_and_batch_split_invariance():
    """Particles never couple: permuting or splitting the batch gives identical rows."""
    spec = make_config(2, n=6)
    csp = O.build_csp(spec)
    x, g = O.initialize_particles(spec, csp, 11, np.arange(6))
    J, Jc, soft, gr = O.cost_and_grad(spec, csp, x, g)
    perm = np.array([3, 0, 5, 1, 4, 2])
    Jp, Jcp, softp, grp = O.cost_and_grad(spec, csp, x[perm], g[perm])
    np.testing.assert_array_equal(Jp, J[perm])
    np.testing.assert_array_equal(grp, gr[perm])
    J2, _, _, gr2 = O.cost_and_grad(spec, csp, x[2:3], g[2:3])
    np.testing.assert_array_equal(J2, J[2:3])
    np.testing.assert_array_equal(gr2, gr[2:3])


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 6, "1s"])
def test_gradient_vs_central_fd(cfg):
    """Autograd gradient of Eq. 2 against central finite differences, excluding
    coordinates whose FD is unstable between h and h/10 (kink neighbourhoods, "1e-4-wide").
    "1s" = config 1 with the self-collision term."""
    selfc = cfg == "1s"
    cfg = 1 if selfc else cfg
    n = 3 if cfg != 4 else 2
    spec = make_config(cfg, n=n)
    spec.self_collision = selfc
    csp = O.build_csp(spec)
    x, g = O.initialize_particles(spec, csp, 100 + cfg, np.arange(n))
    _, _, _, gr = O.cost_and_grad(spec, csp, x, g)

    coords = range(csp.D) if cfg != 4 else np.random.default_rng(0).choice(csp.D, 40, replace=False)

    def fd(h):
        out = np.zeros_like(x)
        for d in coords:
            xp, xm = x.copy(), x.copy()
            xp[:, d] += h
            xm[:, d] -= h
            out[:, d] = (_eval(spec, csp, xp, g)[0] - _eval(spec, csp, xm, g)[0]) / (2 * h)
        return out

    f1, f2 = fd(1e-6), fd(1e-7)
    sel = np.zeros(csp.D, bool)
    sel[list(coords)] = True
    f1, f2, gr = f1[:, sel], f2[:, sel], gr[:, sel]
    scale = np.abs(f1) + 1e-6
    smooth = np.abs(f1 - f2) <= 1e-4 * scale
    assert smooth.mean() > 0.9
    err = np.abs(gr - f1)[smooth]
    assert np.all(err <= 1e-5 * scale[smooth] + 1e-7)


# ---------------------------------------------------------------------------------------------
# Adam (Kingma & Ba) + projection (L11)
# ---------------------------------------------------------------------------------------------
def _toy_csp(D, lr=0.01):
    csp = O.CSP(terms=[], traj_costs=[], goal={}, offsets={}, D=D, grasp_vars=[],
                lo=-np.ones(D) * np.inf, hi=np.ones(D) * np.inf, lr=np.ones(D) * lr)
    spec = make_config(1, n=1)
    return spec, csp


def test_adam_first_step_closed_form_and_zero_gradient():
    """x1 = x0 - lr g / (|g| + eps) at t = 1; zero gradient leaves x unchanged."""
    spec, csp = _toy_csp(5)
    st = O.new_state(np.zeros((1, 5)), np.zeros((1, 0, 3, 4)))
    g = np.array([[1.0, -2.0, 1e-3, 0.0, 1e-9]])
    O.adam_update(spec, csp, st, g)
    np.testing.assert_allclose(st.x[0], -0.01 * g[0] / (np.abs(g[0]) + spec.adam_eps), rtol=1e-12, atol=1e-18)
    assert st.x[0, 3] == 0.0


def test_adam_matches_torch_optim_adam():
    """50 steps with random gradients equal torch.optim.Adam (library routine) in float64."""
    rng = np.random.default_rng(12)
    spec, csp = _toy_csp(7, lr=0.03)
    x0 = rng.normal(size=(3, 7))
    st = O.new_state(x0, np.zeros((3, 0, 3, 4)))
    p = torch.nn.Parameter(torch.tensor(x0, dtype=DT))
    opt = torch.optim.Adam([p], lr=0.03, betas=(spec.beta1, spec.beta2), eps=spec.adam_eps)
    for _ in range(50):
        g = rng.normal(size=(3, 7))
        O.adam_update(spec, csp, st, g)
        p.grad = torch.tensor(g, dtype=DT)
        opt.step()
    np.testing.assert_allclose(st.x, p.detach().numpy(), rtol=1e-12, atol=1e-14)


def test_adam_constant_gradient_and_clamp():
    """Constant gradient for 100 steps moves ~100 lr (within 5 %); clamp to bounds, moments untouched."""
    spec, csp = _toy_csp(2)
    csp.lo = np.array([-np.inf, -0.05])
    csp.hi = np.array([np.inf, np.inf])
    st = O.new_state(np.zeros((1, 2)), np.zeros((1, 0, 3, 4)))
    for _ in range(100):
        O.adam_update(spec, csp, st, np.array([[1.0, 1.0]]))
    assert abs(st.x[0, 0] + 1.0) < 0.05
    assert st.x[0, 1] == -0.05
    assert st.m[0, 1] == st.m[0, 0]


def test_invalid_particles_are_sticky_and_not_updated():
    spec, csp = _toy_csp(2)
    st = O.new_state(np.zeros((2, 2)), np.zeros((2, 0, 3, 4)))
    st.invalid[1] = True
    O.adam_update(spec, csp, st, np.ones((2, 2)))
    assert np.all(st.x[1] == 0.0) and np.all(st.x[0] != 0.0)


# ---------------------------------------------------------------------------------------------
# samplers
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("cfg", [1, 2, 4, 6])
def test_samplers(cfg):
    spec = make_config(cfg, n=512)
    csp = O.build_csp(spec)
    x, g = O.initialize_particles(spec, csp, 77, np.arange(512))
    x2, g2 = O.initialize_particles(spec, csp, 77, np.arange(512))
    assert np.array_equal(x, x2) and np.array_equal(g, g2)                  # determinism
    assert np.all(x >= csp.lo) and np.all(x <= csp.hi)                      # positive density inside bounds
    xs, _ = O.initialize_particles(spec, csp, 77, np.arange(100, 612))
    np.testing.assert_array_equal(xs[:412], x[100:])                         # global-index counters
    for vi, v in enumerate(spec.variables):
        if v.kind == PLACEMENT and not v.const:
            s = spec.surfaces[v.surface]
            o = spec.objects[v.obj]
            if any(a.kind in (PRESS, PRESS_STICK) and a.placement == vi for a in spec.actions):
                o = dataclasses.replace(o, footprint=0.0)          # press poses: whole button face (R8)
            p = x[:, csp.offsets[vi]:csp.offsets[vi] + 4]
            assert np.all(p[:, 2] == s.frame[2])
            c, sn = math.cos(s.frame[3]), math.sin(s.frame[3])
            dx, dy = p[:, 0] - s.frame[0], p[:, 1] - s.frame[1]
            lx, ly = c * dx + sn * dy, -sn * dx + c * dy
            assert np.all(lx >= s.lo[0] + min(o.footprint, (s.hi[0] - s.lo[0]) / 2) - 1e-12)
            assert np.all(lx <= s.hi[0] - min(o.footprint, (s.hi[0] - s.lo[0]) / 2) + 1e-12)
            assert np.all(ly >= s.lo[1] + min(o.footprint, (s.hi[1] - s.lo[1]) / 2) - 1e-12)
    for k in range(g.shape[1]):
        R = g[:, k, :, :3]
        np.testing.assert_allclose(R[:, :, 2], np.tile([0, 0, -1.0], (512, 1)), atol=1e-12)
        yaw = np.arctan2(R[:, 1, 0], R[:, 0, 0])
        h, _ = np.histogram(yaw, bins=16, range=(-math.pi, math.pi))
        assert ((h - 32.0) ** 2 / 32.0).sum() < 37.7
    if cfg == 4:     # knots are the linear interpolation of the motion's endpoint confs
        a = [a for a in spec.actions if a.traj >= 0][1]
        qa = x[:, csp.offsets[a.q1]:csp.offsets[a.q1] + 7]
        qb = x[:, csp.offsets[a.q2]:csp.offsets[a.q2] + 7]
        k2 = x[:, csp.offsets[a.traj] + 7:csp.offsets[a.traj] + 14]
        np.testing.assert_allclose(k2, qa + 0.5 * (qb - qa), atol=1e-12)


# ---------------------------------------------------------------------------------------------
# check counts and best-k
# ---------------------------------------------------------------------------------------------
def test_check_counts_and_best_k_brute_force():
    spec = make_config(1, n=64)
    csp = O.build_csp(spec)
    x, g = O.initialize_particles(spec, csp, 3, np.arange(64))
    st = O.new_state(x, g)
    st.invalid[5] = True
    cls, counts, J, soft, Jc = O.check(spec, csp, st)
    eps = [spec.eps[t.kind] for t in csp.terms]
    for c in range(len(csp.terms)):
        assert counts[c] == sum(1 for i in range(64) if Jc[i, c] <= eps[c])
    assert cls[5] == 2 and counts[-1] == 1
    # force a few classes and ties
    cls = cls.copy()
    cls[[1, 9, 20]] = 0
    soft = soft.copy()
    soft[[1, 9, 20]] = [0.3, 0.1, 0.1]
    gidx = np.arange(64) + 1000
    sel, kc, kcost = O.best_k(cls, J, soft, gidx, 6)
    keys = []
    for i in range(64):
        cost = soft[i] if cls[i] == 0 else (J[i] if cls[i] == 1 else 0.0)
        keys.append((int(cls[i]), cost, gidx[i], i))
    keys.sort()
    assert list(sel) == [k[3] for k in keys[:6]]
    assert list(sel[:3]) == [9, 20, 1]


def test_ik_dls_converges_to_fk_generated_targets():
    """Conditional IK sampler: targets generated by FK (pinned above) are reached; a wrong Jacobian
    column or error sign would stall or diverge."""
    from workloads import panda_robot
    r = panda_robot()
    rng = np.random.default_rng(0)
    qt = rng.uniform(r.joint_lo + 0.3, r.joint_hi - 0.3, (100, 7))
    T = O.forward_kinematics(r, torch.tensor(qt))[:, 8].numpy()
    q0 = np.clip(qt + rng.normal(0, 0.3, (100, 7)), r.joint_lo, r.joint_hi)
    q = O.ik_dls(r, q0, T, 50, 0.1)
    ep, er = O.pose_error(O.forward_kinematics(r, torch.tensor(q))[:, 8], torch.tensor(T))
    assert np.median(ep.numpy()) < 1e-9 and np.median(er.numpy()) < 1e-9
    assert (ep.numpy() < 1e-6).mean() > 0.7
    assert np.all(q >= r.joint_lo) and np.all(q <= r.joint_hi)


def test_ik_initialisation_improves_kin_residuals():
    """InitializeParticles with the IK sampler: Kin residuals drop by orders of magnitude vs uniform confs."""
    spec = make_config(1, n=64)
    csp = O.build_csp(spec)
    x0, g0 = O.initialize_particles(spec, csp, 9, np.arange(64))
    spec.ik_iters = 30
    x1, g1 = O.initialize_particles(spec, csp, 9, np.arange(64))
    assert np.array_equal(g0, g1)
    _, Jc0, _ = _eval(spec, csp, x0, g0)
    _, Jc1, _ = _eval(spec, csp, x1, g1)
    assert np.median(Jc1[:, 2]) < 0.1 * np.median(Jc0[:, 2])
    assert ((Jc1[:, 2] <= 5e-3) & (Jc1[:, 3] <= 0.05)).mean() > 0.25


def test_ik_restarts_keep_first_converged_restart():
    """IK restarts (R6): restart 0 is the single-seed sampler exactly; with 8 restarts the kept conf is the first
    restart that reaches the FK target (checked against FK, pinned above) and far more Kin terms start satisfied;
    restart s draws Philox blocks 2s, 2s+1 of the conf's stream (the same draw the conf sampler makes for s = 0)."""
    from oracle.philox import uniforms
    spec = make_config(3, n=96)
    spec.ik_iters = 20
    csp = O.build_csp(spec)
    gidx = np.arange(96)
    x1, g = O.initialize_particles(spec, csp, 4, gidx)
    spec.ik_seeds = 8
    x8, g8 = O.initialize_particles(spec, csp, 4, gidx)
    assert np.array_equal(g, g8)
    _, Jc1, _ = _eval(spec, csp, x1, g)
    _, Jc8, _ = _eval(spec, csp, x8, g)
    kin = [i for i, t in enumerate(csp.terms) if t.kind in ("KP", "KR")]
    ok1 = np.all(Jc1[:, kin] <= np.array([spec.eps[csp.terms[i].kind] for i in kin]), axis=1)
    ok8 = np.all(Jc8[:, kin] <= np.array([spec.eps[csp.terms[i].kind] for i in kin]), axis=1)
    assert ok8.mean() > 0.5 and ok8.mean() > 5 * max(ok1.mean(), 0.01)
    # first conf of the skeleton: recompute the restarts by hand and check the kept one
    a = [a for a in spec.actions if a.kind == 1][0]           # the first Pick
    off, vi = csp.offsets[a.q1], a.q1
    q0 = spec.robot.joint_lo + uniforms(4, gidx, vi, 7) * (spec.robot.joint_hi - spec.robot.joint_lo)
    pv = spec.variables[a.placement]
    bottom = np.zeros((96, 1, 4))
    bottom[..., 3] = 1.0
    Tt = (O.pose_xyzyaw(torch.as_tensor(np.broadcast_to(pv.value, (96, 4)).copy())) @
          torch.as_tensor(np.concatenate([g[:, 0], bottom], 1))).numpy()
    u = uniforms(4, gidx, vi, 64)
    assert np.array_equal(u[:, :7], uniforms(4, gidx, vi, 7))
    qs = [O.ik_dls(spec.robot, q0 if s == 0 else spec.robot.joint_lo + u[:, 8 * s:8 * s + 7] *
                   (spec.robot.joint_hi - spec.robot.joint_lo), Tt, 20, spec.ik_damping) for s in range(8)]
    errs = [O.ik_errors(spec.robot, q, Tt) for q in qs]
    for i in range(96):
        conv = [s for s in range(8) if errs[s][0][i] <= 1e-3 and errs[s][1][i] <= 1e-3]
        keep = conv[0] if conv else int(np.argmin([errs[s][0][i] + errs[s][1][i] for s in range(8)]))
        assert np.array_equal(x8[i, off:off + 7], qs[keep][i])
    F = O.forward_kinematics(spec.robot, torch.as_tensor(x8[:, off:off + 7]))[:, 8].numpy()
    reached = np.linalg.norm(F[:, :3, 3] - Tt[:, :3, 3], axis=1) <= 1e-3
    assert reached.mean() > 0.8


def test_plan_heuristic_eq5():
    """counts [10, 5] -> H = 7.5; a zero count takes the penalty."""
    assert O.plan_heuristic([10, 5], -100.0) == 7.5
    assert O.plan_heuristic([10, 0], -100.0) == -45.0


def test_self_collision_term():
    """SELF: 0 at the home pose; equals a brute-force loop over the robot's
    sphere pairs on non-adjacent links; emitted after every CF term."""
    from workloads.scenes import Q_HOME
    spec = make_config(1, n=4)
    spec.self_collision = True
    csp = O.build_csp(spec)
    assert [t.kind for t in csp.terms][:5] == ["JL", "CF", "SELF", "KP", "KR"]
    rob = spec.robot
    rng = np.random.default_rng(4)
    q = rng.uniform(rob.joint_lo, rob.joint_hi, (64, 7))
    q[0] = Q_HOME
    x = np.zeros((64, csp.D))
    off = csp.offsets[csp.terms[2].conf[1]]
    x[:, off:off + 7] = q
    g = np.tile(np.eye(3, 4)[None, None], (64, 1, 1, 1))
    _, Jc, _ = _eval(spec, csp, x, g)
    W = O.robot_sphere_centers(rob, O.forward_kinematics(rob, torch.tensor(q))).numpy()
    r = rob.spheres[:, 3]
    ref = np.zeros(64)
    for i in range(len(r)):
        for j in range(i + 1, len(r)):
            if abs(int(rob.sphere_link[i]) - int(rob.sphere_link[j])) >= 2 and (i, j) != (7, 12):
                ref += np.maximum(0.0, r[i] + r[j] - np.linalg.norm(W[:, i] - W[:, j], axis=-1))
    np.testing.assert_allclose(Jc[:, 2], ref, rtol=1e-12, atol=1e-15)
    assert Jc[0, 2] == 0.0 and (ref > 0).mean() > 0.2


def test_smooth_collision_cost_shape():
    """CHOMP-smooth cost: 0 below contact, quadratic up to eta, linear beyond; C^1 at 0
    and eta; the hinge minus eta/2 deep inside."""
    eta = 0.02
    p = torch.tensor([-0.01, 0.0, 0.005, 0.02, 0.05], dtype=DT, requires_grad=True)
    c = O.collision_cost(p, eta, smooth=True)
    np.testing.assert_allclose(c.detach().numpy(), [0.0, 0.0, 0.005 ** 2 / 0.04, 0.01, 0.04], atol=1e-15)
    c.sum().backward()
    np.testing.assert_allclose(p.grad.numpy(), [0.0, 0.0, 0.25, 1.0, 1.0], atol=1e-12)
    np.testing.assert_allclose(O.collision_cost(p.detach(), eta).numpy(), [0, 0, 0.005, 0.02, 0.05], atol=1e-15)


def test_smooth_collision_gradient_vs_fd():
    spec = make_config(2, n=3)
    spec.collision_smooth = True
    spec.eta = 0.02
    spec.self_collision = True
    csp = O.build_csp(spec)
    x, g = O.initialize_particles(spec, csp, 5, np.arange(3))
    _, _, _, gr = O.cost_and_grad(spec, csp, x, g)
    h = 1e-6
    for d in range(0, csp.D, 5):
        xp, xm = x.copy(), x.copy()
        xp[:, d] += h
        xm[:, d] -= h
        fd = (_eval(spec, csp, xp, g)[0] - _eval(spec, csp, xm, g)[0]) / (2 * h)
        np.testing.assert_allclose(gr[:, d], fd, rtol=1e-4, atol=1e-5)


def test_six_dof_grasp_sampler():
    """6-DOF grasps: proper rotations whose approach axis is -z (top) or horizontal into one
    of the four sides, faces roughly uniform; top-down mode unchanged."""
    spec = make_config(1, n=2000)
    spec.objects[0].grasp_mode = 1
    csp = O.build_csp(spec)
    _, g = O.initialize_particles(spec, csp, 3, np.arange(2000))
    R = g[:, 0, :, :3]
    np.testing.assert_allclose(R @ R.transpose(0, 2, 1), np.tile(np.eye(3), (2000, 1, 1)), atol=1e-12)
    np.testing.assert_allclose(np.linalg.det(R), 1.0, atol=1e-12)
    a = R[:, :, 2]
    dirs = np.array([[0, 0, -1], [-1, 0, 0], [1, 0, 0], [0, -1, 0], [0, 1, 0]], float)
    face = np.argmax(a @ dirs.T, axis=1)
    np.testing.assert_allclose(a, dirs[face], atol=1e-12)
    h = np.bincount(face, minlength=5)
    assert ((h - 400.0) ** 2 / 400.0).sum() < 18.5          # chi^2, 4 dof, p = 0.001
    side = face > 0
    np.testing.assert_allclose(g[side, 0, :2, 3], 0.0, atol=1e-15)


# ---------------------------------------------------------------------------------------------
# Stick Button: PressButton / PressButtonStick (R8)
# ---------------------------------------------------------------------------------------------
def test_press_skeleton_terms():
    """PressButton: Kin + ValidPress, hand empty; PressButtonStick: Kin + ValidStickPress with the stick held
    (P:1055-1063).  The robot's CF at a press conf ignores the pressed button; the virtual fingertip is never
    in a scene; the held stick is checked by CP at its press pose, not by CF."""
    spec = make_config(6, n=2)
    csp = O.build_csp(spec)
    kinds = [t.kind for t in csp.terms]
    assert kinds == ["JL", "CF", "KP", "KR", "SS", "PC",              # PressButton(red)
                     "JL", "CF", "KP", "KR",                          # Pick(stick)
                     "JL", "CF", "KP", "KR", "SS", "PC", "CP"]        # PressButtonStick(blue)
    red, blue = spec.surfaces[0].support_obb, spec.surfaces[1].support_obb
    assert csp.terms[1].excl_obb == (red,) and csp.terms[11].excl_obb == (blue,)
    assert csp.terms[7].excl_obb == ()
    for t in csp.terms:
        if t.scene is not None:
            assert 1 not in t.scene                       # fingertip: virtual
    assert 0 in csp.terms[1].scene                        # stick on the table while pressing red
    assert 0 not in csp.terms[11].scene and 0 not in csp.terms[16].scene   # stick held
    assert csp.terms[16].surface == 1 and csp.terms[15].obj == 0
    kinds7 = [t.kind for t in O.build_csp(make_config(7, n=2)).terms]
    assert kinds7 == ["JL", "CF", "KP", "KR", "SS", "PC"] * 2


def _rect_dist(px, py, lo, hi):
    """Euclidean distance from a point to an axis-aligned rectangle (projection by clipping)."""
    cx, cy = np.clip(px, lo[0], hi[0]), np.clip(py, lo[1], hi[1])
    return math.hypot(px - cx, py - cy)


def test_press_contact_closed_form():
    """PC = min over the pressing object's spheres of the distance from the sphere centre's xy to the button
    face (projection by clipping), SS = |z_bottom - z_top|; random fingertip and stick press poses."""
    spec = make_config(6, n=1)
    csp = O.build_csp(spec)
    rng = np.random.default_rng(3)
    x0, g = O.initialize_particles(spec, csp, 1, np.arange(1))
    off_r = csp.offsets[[i for i, v in enumerate(spec.variables) if v.name == "press_red"][0]]
    off_b = csp.offsets[[i for i, v in enumerate(spec.variables) if v.name == "press_blue_stick"][0]]
    sr, sb = spec.surfaces[0], spec.surfaces[1]
    for _ in range(20):
        x = x0.copy()
        pr = np.array([sr.frame[0] + rng.uniform(-0.06, 0.06), sr.frame[1] + rng.uniform(-0.06, 0.06),
                       sr.frame[2] + rng.uniform(-0.01, 0.01), rng.uniform(-4, 4)])
        pb = np.array([sb.frame[0] + rng.uniform(-0.3, 0.3), sb.frame[1] + rng.uniform(-0.3, 0.3),
                       sb.frame[2] + rng.uniform(-0.01, 0.01), rng.uniform(-4, 4)])
        x[0, off_r:off_r + 4] = pr
        x[0, off_b:off_b + 4] = pb
        _, Jc, _ = _eval(spec, csp, x, g)
        # fingertip: one sphere on the frame's z axis
        assert Jc[0, 4] == pytest.approx(abs(pr[2] - sr.frame[2]), abs=1e-15)
        assert Jc[0, 5] == pytest.approx(_rect_dist(pr[0] - sr.frame[0], pr[1] - sr.frame[1], sr.lo, sr.hi),
                                         rel=1e-12, abs=1e-15)
        st = spec.objects[0]
        c, sn = math.cos(pb[3]), math.sin(pb[3])
        d = min(_rect_dist(pb[0] + c * sp[0] - sn * sp[1] - sb.frame[0], pb[1] + sn * sp[0] + c * sp[1] - sb.frame[1],
                           sb.lo, sb.hi) for sp in st.spheres)
        assert Jc[0, 14] == pytest.approx(abs(pb[2] - sb.frame[2]), abs=1e-15)
        assert Jc[0, 15] == pytest.approx(d, rel=1e-12, abs=1e-15)


def test_constructed_press_particle_satisfies_press_terms():
    """Fingertip press pose inside the red face at its height; conf by IK onto T(p) T(g): SS, PC
    exactly 0 and the Kin residuals at IK precision, so ValidPress and Kin hold (Eq. 3)."""
    spec = make_config(6, n=4)
    csp = O.build_csp(spec)
    x, g = O.initialize_particles(spec, csp, 9, np.arange(4))
    vi = [i for i, v in enumerate(spec.variables) if v.name == "press_red"][0]
    qi = [i for i, v in enumerate(spec.variables) if v.name == "q_press_red"][0]
    s = spec.surfaces[0]
    rng = np.random.default_rng(0)
    p = np.stack([s.frame[0] + rng.uniform(-0.015, 0.015, 4), s.frame[1] + rng.uniform(-0.015, 0.015, 4),
                  np.full(4, s.frame[2]), rng.uniform(-3, 3, 4)], 1)
    x[:, csp.offsets[vi]:csp.offsets[vi] + 4] = p
    Tg = np.concatenate([g[:, 0], np.tile([[[0, 0, 0, 1.0]]], (4, 1, 1))], 1)
    Tt = (O.pose_xyzyaw(torch.as_tensor(p)) @ torch.as_tensor(Tg)).numpy()
    q0 = np.tile(make_config(1).variables[0].value, (4, 1))
    x[:, csp.offsets[qi]:csp.offsets[qi] + 7] = O.ik_dls(spec.robot, q0, Tt, 200, 0.05)
    _, Jc, _ = _eval(spec, csp, x, g)
    assert np.all(Jc[:, 4] == 0.0) and np.all(Jc[:, 5] == 0.0)
    assert np.all(Jc[:, 2] <= 1e-6) and np.all(Jc[:, 3] <= 1e-6)
    tol = np.array([spec.eps[k] for k in ("KP", "KR", "SS", "PC")])
    assert np.all(Jc[:, 2:6] <= tol)


def test_stick_grasp_range():
    """Top-down stick grasps: TCP anywhere along the stick (|gx| <= grasp_xy) and on its axis (|gy| <= grasp_y)."""
    spec = make_config(6, n=1000)
    csp = O.build_csp(spec)
    _, g = O.initialize_particles(spec, csp, 4, np.arange(1000))
    st = spec.objects[0]
    k = csp.grasp_vars.index([i for i, v in enumerate(spec.variables) if v.name == "g_stick"][0])
    assert np.all(np.abs(g[:, k, 0, 3]) <= st.grasp_xy) and np.abs(g[:, k, 0, 3]).max() > 0.9 * st.grasp_xy
    assert np.all(np.abs(g[:, k, 1, 3]) <= st.grasp_y) and np.abs(g[:, k, 1, 3]).max() > 0.9 * st.grasp_y
    kf = csp.grasp_vars.index([i for i, v in enumerate(spec.variables) if v.name == "g_fingertip"][0])
    np.testing.assert_array_equal(g[:, kf, :, 3], 0.0)
