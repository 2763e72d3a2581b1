"""CPU-side checks of the C ABI library: it builds/loads, exports every symbol include/tamp.h declares,
the ctypes layout matches, and the host-side skeleton compiler accepts the five configs and rejects bad
descriptors (no GPU needed: tamp_query_workspace only compiles)."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

import paper_2411_11833_b200 as pkg
from paper_2411_11833_b200 import build as b
from paper_2411_11833_b200 import tamp as T
from workloads import make_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    b.build()
    return pkg.load()


def test_exports_every_declared_symbol(lib):
    hdr = open(os.path.join(ROOT, "include", "tamp.h")).read()
    declared = set(re.findall(r"\b(tamp_[a-z_0-9]+)\s*\(", hdr))
    assert len(declared) >= 15
    cdll = ctypes.CDLL(T.LIB_PATH)
    for name in sorted(declared):
        assert hasattr(cdll, name), f"libtamp.so does not export {name}"
    assert set(T.EXPORTS) <= declared


def test_struct_layout_matches(lib):
    assert lib.tamp_sizeof_desc() == ctypes.sizeof(T.ProblemDesc)
    assert lib.tamp_sizeof_info() == ctypes.sizeof(T.Info)
    assert lib.tamp_abi_version() == T.ABI_VERSION


def _query(lib, desc, n):
    nb = ctypes.c_size_t()
    st = lib.tamp_query_workspace(ctypes.byref(desc), n, ctypes.byref(nb))
    return st, nb.value, lib.tamp_last_error().decode()


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5, 6, 7])
def test_compiler_accepts_configs(lib, cfg):
    spec = make_config(cfg, n=16)
    st, nb, msg = _query(lib, T.build_desc(spec), 1000)
    assert st == 0, msg
    assert nb > 1000 * 3 * 4


def test_compiler_rejects_bad_descriptors(lib):
    spec = make_config(1, n=4)
    d = T.build_desc(spec)
    d.robot.joint_lo[2] = d.robot.joint_hi[2] + 1
    st, _, msg = _query(lib, d, 10)
    assert st == 1 and "joint_lo" in msg
    d = T.build_desc(spec)
    d.lam[3] = 0.0
    st, _, msg = _query(lib, d, 10)
    assert st == 1 and "lambda" in msg
    d = T.build_desc(spec)
    d.obb[0].half[1] = -1
    assert _query(lib, d, 10)[0] == 1
    d = T.build_desc(spec)
    d.abi_version = 99
    assert _query(lib, d, 10)[0] == 1
    d = T.build_desc(spec)
    d.action[1].placement = d.action[3].placement      # Pick from a placement the object is not at
    st, _, msg = _query(lib, d, 10)
    assert st == 1 and "Pick" in msg
    d = T.build_desc(spec)
    d.robot.n_spheres = 33
    assert _query(lib, d, 10)[0] == 5
    assert _query(lib, T.build_desc(spec), 0)[0] == 1


def test_compiler_rejects_bad_press_actions(lib):
    """PressButton needs an empty hand and the virtual fingertip; PressButtonStick needs the stick held;
    Pick of a virtual object is rejected (P:1055-1063 preconditions)."""
    spec = make_config(6, n=4)
    assert _query(lib, T.build_desc(spec), 10)[0] == 0
    d = T.build_desc(spec)
    d.action[1].obj = 0                                 # PressButton with the stick (not virtual)
    st, _, msg = _query(lib, d, 10)
    assert st == 1 and "grasp" in msg or "virtual" in msg
    d = T.build_desc(spec)
    d.action[5].kind = 4                                # PressButton while holding the stick
    st, _, msg = _query(lib, d, 10)
    assert st == 1 and "hand not empty" in msg
    d = T.build_desc(spec)
    d.action[4].kind = 0                                # no MoveHold: fine; drop the Pick -> stick not held
    d.action[3].kind = 0
    d.action[3].q2 = d.action[3].q1
    st, _, msg = _query(lib, d, 10)
    assert st == 1 and "not held" in msg
    d = T.build_desc(spec)
    d.action[3].obj = 1                                 # Pick the virtual fingertip
    d.action[3].grasp = 2
    st, _, msg = _query(lib, d, 10)
    assert st == 1


def test_product_path_fails_loudly_without_library(tmp_path):
    with pytest.raises(RuntimeError):
        T._lib_backup = T._lib
        T._lib = None
        try:
            T.load(str(tmp_path / "missing.so"))
        finally:
            T._lib = T._lib_backup


def test_plan_heuristic_matches_oracle(lib):
    from oracle import tamp_oracle as O
    rng = np.random.default_rng(0)
    for _ in range(20):
        c = rng.integers(0, 5, size=rng.integers(1, 40))
        assert pkg.plan_heuristic(c, len(c), -1e3) == pytest.approx(O.plan_heuristic(c, -1e3), rel=1e-12)
    assert pkg.plan_heuristic([10, 5, 0, 0], 2, -1.0) == 7.5


def test_obb_rotation_validated(lib):
    """tamp_obb_desc.rot: all zeros -> Rz(yaw); a rotation matrix is accepted; a non-orthonormal or reflecting
    matrix is TAMP_E_INVALID (include/tamp.h)."""
    spec = make_config(1, n=4)
    d = T.build_desc(spec)
    c, s = math.cos(0.3), math.sin(0.3)
    for k, v in enumerate([1, 0, 0, 0, c, -s, 0, s, c]):
        d.obb[0].rot[k] = v
    assert _query(lib, d, 10)[0] == 0
    d.obb[0].rot[0] = 1.1
    st, _, msg = _query(lib, d, 10)
    assert st == 1 and "rot" in msg
    for k, v in enumerate([-1, 0, 0, 0, 1, 0, 0, 0, 1]):       # det -1
        d.obb[0].rot[k] = v
    assert _query(lib, d, 10)[0] == 1


def test_obb_extent_bound(lib):
    """Boxes must lie within 100 m of the origin (|c_k| + h_k <= 100): the kernels' reject test for axis-aligned
    boxes grows the corners by 2e-5 m, which covers fp32 rounding only up to that scale (TAMP_E_UNSUPPORTED = 5
    beyond, include/tamp.h)."""
    spec = make_config(1, n=4)
    d = T.build_desc(spec)
    d.obb[0].center[0] = 99.0
    assert _query(lib, d, 10)[0] == 0
    d.obb[0].center[0] = 101.0
    st, _, msg = _query(lib, d, 10)
    assert st == 5 and "100 m" in msg
