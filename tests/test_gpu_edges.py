"""GPU parity at the method's degenerate points, through the C ABI against the oracle.

* rotation error theta within 1e-3 of pi and at pi (L4: the atan2 form of the geodesic angle; cost only, the
  gradient direction is not unique there);
* coincident sphere centres (L13: hinge r_a + r_b, zero gradient from that pair);
* a residual exactly at its tolerance, J_c = eps_c, is satisfying, one float32 ulp beyond is not (Eq. 3 "<=",
  L21).
"""
import copy
import math

import numpy as np
import pytest
import torch

from oracle import tamp_oracle as O
from paper_2411_11833_b200 import TampContext
from paper_2411_11833_b200 import build as b
from workloads import make_config
from workloads.scenes import PLACEMENT

from parity_utils import COST_ATOL, COST_RTOL, grad_ok, to_ctx_grasp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    b.build()
    torch.cuda.set_device(0)


def _ctx(spec, x32, g32):
    n = x32.shape[0]
    ctx = TampContext(spec, n)
    ctx.set_state(torch.from_numpy(x32).cuda(), grasp=to_ctx_grasp(g32).cuda())
    return ctx


def test_rotation_error_near_pi_cost():
    """Constructed satisfying pick-place particles (T(g) := T(p0)^-1 FK(q)) with the place target's yaw turned by
    psi = pi - {1e-3, 3e-4, 1e-4, 0}: R_ee^T R* = R_g^T Rz(psi) R_g, so KR = psi exactly in the oracle; the GPU's
    KR and every other J_c agree to the cost tolerance."""
    from test_oracle_csp import _clear_pickplace, satisfying_particle
    spec = _clear_pickplace()
    csp = O.build_csp(spec)
    rng = np.random.default_rng(11)
    offs = [math.pi - 1e-3, math.pi - 3e-4, math.pi - 1e-4, math.pi, -(math.pi - 1e-3)]
    xs, gs = [], []
    for d in offs:
        x, Tg = satisfying_particle(spec, csp, rng)
        x[csp.offsets[csp.terms[8].placement] + 3] += d
        xs.append(x)
        gs.append(Tg[None])
    x32, g32 = np.array(xs, np.float32), np.array(gs, np.float32)
    ctx = _ctx(spec, x32, g32)
    J, soft, Jc, _ = (t.cpu().numpy() for t in ctx.eval())
    Jo, Jco, softo, _ = O.cost_and_grad(spec, csp, x32.astype(np.float64), g32.astype(np.float64))
    np.testing.assert_allclose(Jco[:, 7], np.abs(np.float32(offs)).astype(np.float64), atol=2e-6)
    np.testing.assert_allclose(Jc, Jco, rtol=COST_RTOL, atol=COST_ATOL)
    np.testing.assert_allclose(J, Jo, rtol=COST_RTOL, atol=COST_ATOL)


def test_coincident_sphere_centres():
    """Config 2 with both obstructors placed at exactly the same pose: every sphere of A coincides with the same
    sphere of B.  The CFreePlace hinge of such a pair is r_a + r_b and its gradient is 0 (L13); the other pairs
    between the two are ordinary.  Cost, per-term costs and gradient agree with the oracle."""
    n = 8
    spec = make_config(2, n=n)
    csp = O.build_csp(spec)
    x, g = O.initialize_particles(spec, csp, 91, np.arange(n))
    pa, pb = [vi for vi, v in enumerate(spec.variables) if v.kind == PLACEMENT and not v.const][:2]
    x[:, csp.offsets[pb]:csp.offsets[pb] + 4] = x[:, csp.offsets[pa]:csp.offsets[pa] + 4]
    x32, g32 = x.astype(np.float32), g.astype(np.float32)
    ctx = _ctx(spec, x32, g32)
    J, soft, Jc, grad = (t.cpu().numpy() for t in ctx.eval())
    Jo, Jco, softo, grado = O.cost_and_grad(spec, csp, x32.astype(np.float64), g32.astype(np.float64))
    i_cp = [i for i, t in enumerate(csp.terms) if t.kind == "CP"][1]       # obstructor B placed next to A
    r = spec.objects[1].spheres[:, 3]
    assert np.all(Jco[:, i_cp] >= 2 * r.sum() - 1e-7)                       # 8 coincident pairs at r_a + r_b
    np.testing.assert_allclose(Jc, Jco, rtol=COST_RTOL, atol=COST_ATOL)
    np.testing.assert_allclose(J, Jo, rtol=COST_RTOL, atol=COST_ATOL)
    assert grad_ok(grad, grado).all()


def test_residual_exactly_at_tolerance_is_satisfying():
    """StablePlace support |z_bottom - z_top| = eps_SS exactly (the region's surface lowered by eps_SS, a float32
    number, the block at z = 0) is satisfying on the GPU as in the oracle ("5 mm exactly is satisfying");
    lowering the surface by one more float32 ulp makes that term, and the particle, unsatisfied."""
    from test_oracle_csp import _clear_pickplace, satisfying_particle
    spec = _clear_pickplace()
    csp = O.build_csp(spec)
    rng = np.random.default_rng(12)
    x, Tg = satisfying_particle(spec, csp, rng)
    x32 = x[None].astype(np.float32)
    g32 = Tg[None, None].astype(np.float32)
    e = np.float32(spec.eps["SS"])
    for z_top, sat in ((-e, True), (-np.nextafter(e, np.float32(1.0)), False)):
        s2 = copy.deepcopy(spec)
        s2.surfaces[0].frame[2] = float(z_top)
        ctx = _ctx(s2, x32, g32)
        cls = torch.empty(1, dtype=torch.uint8, device="cuda")
        counts, _ = ctx.check(cls=cls)
        counts = counts.cpu().numpy()
        cls_o, counts_o, _, _, Jc_o = O.check(s2, csp, O.new_state(x32.astype(np.float64), g32.astype(np.float64)))
        assert (cls.cpu().numpy()[0] == 0) == sat and (cls_o[0] == 0) == sat
        assert counts[8] == (1 if sat else 0) and counts_o[8] == counts[8]
        np.testing.assert_array_equal(counts, counts_o)


def _tilted_scene(cfg, n):
    """Config `cfg` with two fully rotated boxes where the arm and the objects move (P:489 oriented boxes): a slab
    tilted 35 degrees about x over the work area and a box turned about an oblique axis beside it."""
    from scipy.spatial.transform import Rotation
    from workloads.scenes import OBB
    from workloads.scenes import _f32
    spec = make_config(cfg, n=n)
    R1 = Rotation.from_euler("x", 35, degrees=True).as_matrix()
    R2 = Rotation.from_rotvec(0.8 * np.array([0.3, -0.5, 0.81]) / np.linalg.norm([0.3, -0.5, 0.81])).as_matrix()
    spec.obbs = spec.obbs + [_f32(OBB(np.array([0.45, 0.05, 0.30]), 0.0, np.array([0.12, 0.15, 0.02]), "slab", R1)),
                             _f32(OBB(np.array([0.35, -0.25, 0.15]), 0.0, np.array([0.05, 0.08, 0.10]), "tilt", R2))]
    return spec


@pytest.mark.parametrize("cfg,lanes", [(2, 8), (2, 4), (2, 16), (1, 1), (4, 16), (3, 8)])
def test_tilted_boxes_cost_gradient_and_step(cfg, lanes):
    """Full-orientation OBBs through the C ABI (tamp_obb_desc.rot): per-term costs, gradients and one Adam step
    against the oracle on every mapping (serial included)."""
    from parity_utils import STEP_RTOL, kink_mask
    n = 97 if cfg != 4 else 40
    spec = _tilted_scene(cfg, n)
    csp = O.build_csp(spec)
    x, g = O.initialize_particles(spec, csp, 70 + cfg, np.arange(n))
    x32, g32 = x.astype(np.float32), g.astype(np.float32)
    ctx = TampContext(spec, n, n_global=1000, lanes_per_particle=lanes)
    ctx.set_state(torch.from_numpy(x32).cuda(), grasp=to_ctx_grasp(g32).cuda())
    J, soft, Jc, grad = (t.cpu().numpy() for t in ctx.eval())
    Jo, Jco, softo, grado = O.cost_and_grad(spec, csp, x32.astype(np.float64), g32.astype(np.float64))
    # the tilted boxes are hit (otherwise this tests nothing)
    cf = [i for i, t in enumerate(csp.terms) if t.kind in ("CF", "CP")]
    spec0 = make_config(cfg, n=n)
    _, Jc0, _ = O.evaluate(spec0, O.build_csp(spec0), torch.as_tensor(x32.astype(np.float64)),
                           torch.as_tensor(g32.astype(np.float64)))
    assert (Jco[:, cf] > Jc0.detach().numpy()[:, cf] + 1e-6).any(axis=1).mean() > 0.1
    np.testing.assert_allclose(Jc, Jco, rtol=COST_RTOL, atol=COST_ATOL)
    np.testing.assert_allclose(J, Jo, rtol=COST_RTOL, atol=COST_ATOL)
    ok = grad_ok(grad, grado)
    kinks = kink_mask(spec, csp, x32.astype(np.float64), g32.astype(np.float64), grado, np.random.default_rng(0)) \
        if not ok.all() else ~ok
    assert np.all(ok | kinks) and kinks.mean() <= 0.1
    ctx.optimize(1)
    x1 = ctx.get_state()["x"].cpu().numpy()
    so = O.new_state(x32.astype(np.float64), g32.astype(np.float64))
    O.optimize(spec, csp, so, 1, 1.0 / 1000)
    unstable = np.abs(grado) < 1e-4 * np.abs(grado).max(axis=1, keepdims=True)
    close = np.abs(x1 - so.x) <= STEP_RTOL * (np.abs(so.x) + csp.lr[None, :])
    assert np.all(close | unstable | kinks[:, None])


def test_bench_json_line_contract():
    """bench.py (a short run) prints one JSON line with the driver's keys: metric / value / unit / n_gpus / steps /
    warmup / ms_per_step / higher_is_better / scaling / dtype / data / config.workload, plus roofline (bound,
    achieved, peak, unit, frac, traffic), e2e (value, unit, h2d / d2h bytes), gpu_launches > 0, clocks, repeats."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--config", "1", "--n", "512", "--steps", "2",
                        "--warmup", "3", "--repeats", "2", "--no-extra", "--no-cpu-baseline", "--no-ttfs"],
                       capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks", "repeats"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["config"]["workload"].startswith("config1")
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"], k
    assert len(d["repeats"]["values"]) == 2


def test_bench_collective_path_one_rank():
    """bench.py --dist: torch.distributed with the NCCL backend for one rank -- the overlapped C1 all-reduce on the
    side stream, the C2 all-gather and the K5 merge run on the GPU and the line reports the overlapped all-reduce."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MASTER_PORT="29611")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--dist", "--config", "2", "--n", "1024",
                        "--steps", "2", "--warmup", "3", "--repeats", "1", "--no-extra", "--no-cpu-baseline", "--no-ttfs"],
                       capture_output=True, text=True, timeout=600, cwd=root, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    d = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    assert d["n_gpus"] == 1 and d["value"] > 0
    assert "overlapped" in d["config"]["allreduce"]


@pytest.mark.parametrize("lanes,single_box", [(8, False), (8, True), (1, True)])
def test_box_reject_at_reach_boundary(lanes, single_box):
    """The kernels skip a sphere's exact box test when a cheaper reject test says it cannot reach the box (for
    axis-aligned boxes: the corner form with grown corners, obb_reach_corner_pair).  A small axis-aligned box is
    placed against the robot sphere that reaches farthest along +x at the pick configuration, so that the sphere
    penetrates it by d in {3e-5, 1e-5, 2e-6, 0, -2e-6, -1e-5} m: the CF hinge of that configuration equals the
    oracle's (which grows by d for d > 0) to 2e-7.  single_box: the box is the only one (the serial mapping's
    one-box path; the region then has no support box)."""
    from workloads.scenes import OBB
    from workloads.scenes import _f32
    base = make_config(1, n=1)
    csp0 = O.build_csp(base)
    x, g = O.initialize_particles(base, csp0, 5, np.arange(1))
    i_cf = [i for i, t in enumerate(csp0.terms) if t.kind == "CF"][0]
    qo = csp0.offsets[csp0.terms[i_cf].conf[1]]       # conf = ("var", variable index)
    q = torch.tensor(x[:, qo:qo + 7])
    W = O.robot_sphere_centers(base.robot, O.forward_kinematics(base.robot, q))[0].numpy()
    r = base.robot.spheres[:, 3] + base.eta
    s = int(np.argmax(W[:, 0] + r))
    vals = []
    for d in (3e-5, 1e-5, 2e-6, 0.0, -2e-6, -1e-5):
        spec = copy.deepcopy(base)
        h = 0.01
        box = _f32(OBB(np.array([W[s, 0] + r[s] - d + h, W[s, 1], W[s, 2]]), 0.0, np.array([h, h, h]), "probe"))
        if single_box:
            spec.obbs = [box]
            for sf in spec.surfaces:
                sf.support_obb = -1
        else:
            spec.obbs = spec.obbs + [box]
        csp = O.build_csp(spec)
        x32, g32 = x.astype(np.float32), g.astype(np.float32)
        ctx = TampContext(spec, 1, lanes_per_particle=lanes)
        ctx.set_state(torch.from_numpy(x32).cuda(), grasp=to_ctx_grasp(g32).cuda())
        _, _, Jc, _ = (t.cpu().numpy() for t in ctx.eval())
        _, Jco, _, _ = O.cost_and_grad(spec, csp, x32.astype(np.float64), g32.astype(np.float64))
        np.testing.assert_allclose(Jc[0, i_cf], Jco[0, i_cf], rtol=1e-5, atol=2e-7)
        vals.append(Jco[0, i_cf])
    # the construction works: the oracle's hinge grows with the penetration (by 2e-5 from d = 1e-5 to 3e-5)
    assert abs((vals[0] - vals[1]) - 2e-5) < 2e-6 and vals[1] > vals[2] > vals[3] - 1e-9
