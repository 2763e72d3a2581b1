"""The Tetris skeletons are feasible by construction: a hand-constructed particle (tests/constructed.py,
written to tests/golden/tetris_satisfying_cfg{3,4}.npz by tools/make_tetris_fixtures.py with the oracle only) puts the
pieces on an exact tiling of the goal grid, with exact IK confs and collision-free confs / knots, and satisfies every
hard term of Eq. 3 under the tolerances of P:1130-1135 -- in the oracle (CPU) and through the C ABI (GPU)."""
import os

import numpy as np
import pytest
import torch

from oracle import tamp_oracle as O
from workloads import make_config
from workloads.scenes import CELL

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _fixture(cfg):
    f = np.load(os.path.join(GOLDEN, f"tetris_satisfying_cfg{cfg}.npz"))
    return f["x"], f["grasps"], int(f["W"]), int(f["H"]), [str(s) for s in f["shapes"]]


@pytest.mark.parametrize("cfg", [3, 4])
def test_constructed_tetris_particle_is_an_exact_tiling(cfg):
    """The placed pieces' cube centres (two spheres per 4 cm cube) land one-to-one on the cell centres of the W x H
    grid centred in the goal region, at the table height (z = 0, yaw a multiple of pi/2)."""
    x, G, W, H, shapes = _fixture(cfg)
    spec = make_config(cfg, n=1)
    csp = O.build_csp(spec)
    sf = [s for s in spec.surfaces if s.name == "tetris_region"][0]
    centres = []
    for a in spec.actions:
        if a.kind == 3:                      # Place
            p = x[csp.offsets[a.placement]:csp.offsets[a.placement] + 4]
            assert p[2] == pytest.approx(sf.frame[2], abs=1e-12)
            assert (p[3] / (np.pi / 2)) == pytest.approx(round(p[3] / (np.pi / 2)), abs=1e-9)
            T = O.pose_xyzyaw(torch.tensor(p)).numpy()
            sph = spec.objects[a.obj].spheres
            w = (T[:3, :3] @ sph[:, :3].T).T + T[:3, 3]
            centres += [w[k, :2] for k in range(0, len(sph), 2)]
    cells = np.rint((np.array(centres) - [sf.frame[0], sf.frame[1]]) / CELL + [(W - 1) / 2, (H - 1) / 2])
    np.testing.assert_allclose((cells - [(W - 1) / 2, (H - 1) / 2]) * CELL + [sf.frame[0], sf.frame[1]],
                               np.array(centres), atol=1e-6)
    assert sorted(map(tuple, cells.astype(int))) == [(i, j) for i in range(W) for j in range(H)]


@pytest.mark.parametrize("cfg", [3, 4])
def test_constructed_tetris_particle_satisfies_eq3_in_the_oracle(cfg):
    """Class 0: every collision / bounds / support / containment term is exactly 0; the Kin residuals are rounding
    (config 3) or at most a fifth of their tolerances (config 4, whose last pick is at the arm's reach)."""
    x, G, *_ = _fixture(cfg)
    spec = make_config(cfg, n=1)
    csp = O.build_csp(spec)
    cls, counts, J, soft, Jc = O.check(spec, csp, O.new_state(x[None], G[None]))
    assert cls[0] == 0 and counts[-2] == 1
    kin = np.array([t.kind in ("KP", "KR") for t in csp.terms])
    eps = np.array([spec.eps[t.kind] for t in csp.terms])
    assert np.all(Jc[0, ~kin] == 0.0)
    assert np.all(Jc[0, kin] <= (1e-6 if cfg == 3 else 0.2 * eps[kin]))


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,lanes", [(3, 8), (3, 4), (4, 16), (4, 8)])
def test_constructed_tetris_particle_is_class0_on_the_gpu(cfg, lanes):
    """The same particle (fp32) among 47 sampled ones through tamp_check_satisfied: class 0 on the GPU, the same
    classes and per-term counts as the oracle's check of the fp32 inputs; best-k ranks it first (the only satisfying
    particle; key = its soft cost)."""
    from paper_2411_11833_b200 import TampContext, decode_records
    from paper_2411_11833_b200 import build as b
    from parity_utils import to_ctx_grasp
    b.build()
    torch.cuda.set_device(0)
    x, G, *_ = _fixture(cfg)
    n = 48
    spec = make_config(cfg, n=n)
    csp = O.build_csp(spec)
    xs, gs = O.initialize_particles(spec, csp, 5, np.arange(n))
    xs[17], gs[17] = x, G
    x32, g32 = xs.astype(np.float32), gs.astype(np.float32)
    ctx = TampContext(spec, n, lanes_per_particle=lanes)
    ctx.set_state(torch.from_numpy(x32).cuda(), grasp=to_ctx_grasp(g32).cuda())
    cls = torch.empty(n, dtype=torch.uint8, device="cuda")
    counts, _ = ctx.check(cls=cls)
    cls_o, counts_o, _, soft_o, _ = O.check(spec, csp, O.new_state(x32.astype(np.float64), g32.astype(np.float64)))
    assert cls_o[17] == 0 and cls.cpu().numpy()[17] == 0
    np.testing.assert_array_equal(cls.cpu().numpy(), cls_o)
    np.testing.assert_array_equal(counts.cpu().numpy(), counts_o)
    c, cost, gidx, _ = decode_records(ctx.best_k(1))
    assert c[0] == 0 and gidx[0] == 17
    assert cost[0] == pytest.approx(soft_o[17], rel=1e-4, abs=1e-6)
