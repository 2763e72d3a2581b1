#!/usr/bin/env python
"""Write tests/golden/tetris_satisfying_cfg{3,4}.npz: a hand-constructed satisfying particle of the Tetris skeletons
(tests/constructed.py: exact tiling of the goal grid, exact IK, collision-free confs and knots), built and checked
with the oracle only ("feasible by construction").  Deterministic (seeded)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from oracle import tamp_oracle as O  # noqa: E402
from workloads import make_config  # noqa: E402
from constructed import satisfying_tetris  # noqa: E402

CASES = {3: (4, 4, ["I", "L", "O", "J"]), 4: (6, 4, ["I", "L", "O", "J", "I", "I"])}
IK_TOL = {3: (1e-7, 1e-7), 4: (1e-3, 1e-2)}     # config 4: its last piece's pick is at the arm's reach

for cfg in [int(a) for a in sys.argv[1:]] or [3, 4]:
    W, H, shapes = CASES[cfg]
    t0 = time.time()
    spec = make_config(cfg, n=1)
    csp = O.build_csp(spec)
    x, G = satisfying_tetris(spec, csp, np.random.default_rng(cfg), W, H, shapes, ik_tol=IK_TOL[cfg])
    cls, counts, J, soft, Jc = O.check(spec, csp, O.new_state(x[None], G[None]))
    assert cls[0] == 0, "constructed particle is not satisfying"
    path = os.path.join(ROOT, "tests", "golden", f"tetris_satisfying_cfg{cfg}.npz")
    np.savez(path, x=x, grasps=G, W=W, H=H, shapes=np.array(shapes))
    print(f"config {cfg}: class 0, soft {soft[0]:.6f}, max Jc {Jc.max():.3g}, {time.time() - t0:.0f} s -> {path}")
