"""Thin Python binding of libtamp (include/tamp.h): ctypes marshalling only.

Every step of the hot path runs in the CUDA kernels of libtamp.so; PyTorch provides device memory
(the workspace and output tensors), the CUDA stream and, in bench.py, torch.distributed.  There is
no CPU fallback: if libtamp.so is missing or fails to load, `load()` raises.
"""
from __future__ import annotations

import ctypes
import math
import os
from typing import Optional

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtamp.so")

# ---- limits / enums (include/tamp.h) ----
ABI_VERSION = 4
NJ = 7
MAX_ROBOT_SPHERES = 32
MAX_OBB = 16
MAX_OBJECTS = 8
MAX_OBJ_SPHERES = 8
MAX_SURFACES = 8
MAX_VARS = 96
MAX_ACTIONS = 64
MAX_GOAL = 8
MAX_TERMS = 256
N_TERM_KINDS = 9
TERM_NAMES = ("JL", "CF", "KP", "KR", "SS", "SC", "CP", "SELF", "PC")
STATUS = {0: "OK", 1: "E_INVALID", 2: "E_CUDA", 3: "E_NOMEM", 4: "E_STATE", 5: "E_UNSUPPORTED"}

F = ctypes.c_float
I32 = ctypes.c_int32
I64 = ctypes.c_int64


class RobotDesc(ctypes.Structure):
    _fields_ = [("dh", F * 3 * NJ), ("flange_d", F), ("tcp_yaw", F), ("tcp_d", F), ("base", F * 4),
                ("joint_lo", F * NJ), ("joint_hi", F * NJ), ("n_spheres", I32),
                ("sphere", F * 4 * MAX_ROBOT_SPHERES), ("sphere_link", I32 * MAX_ROBOT_SPHERES),
                ("self_mask", ctypes.c_uint32 * MAX_ROBOT_SPHERES)]


class ObbDesc(ctypes.Structure):
    _fields_ = [("center", F * 3), ("yaw", F), ("half", F * 3), ("rot", F * 9)]


class ObjectDesc(ctypes.Structure):
    _fields_ = [("n_spheres", I32), ("sphere", F * 4 * MAX_OBJ_SPHERES), ("footprint", F), ("grasp_xy", F),
                ("grasp_z", F), ("grasp_mode", I32), ("grasp_y", F)]


class SurfaceDesc(ctypes.Structure):
    _fields_ = [("frame", F * 4), ("lo", F * 2), ("hi", F * 2), ("support_obb", I32), ("support_obj", I32)]


class VarDesc(ctypes.Structure):
    _fields_ = [("kind", I32), ("is_const", I32), ("obj", I32), ("surface", I32), ("n_knots", I32),
                ("value", F * 7), ("lo", F * 4), ("hi", F * 4), ("rng_stream", ctypes.c_uint32)]


class ActionDesc(ctypes.Structure):
    _fields_ = [("kind", I32), ("obj", I32), ("grasp", I32), ("placement", I32), ("surface", I32),
                ("q1", I32), ("q2", I32), ("traj", I32)]


class ProblemDesc(ctypes.Structure):
    _fields_ = [("abi_version", I32), ("robot", RobotDesc),
                ("n_obb", I32), ("obb", ObbDesc * MAX_OBB),
                ("n_objects", I32), ("object", ObjectDesc * MAX_OBJECTS),
                ("n_surfaces", I32), ("surface", SurfaceDesc * MAX_SURFACES),
                ("n_vars", I32), ("var", VarDesc * MAX_VARS),
                ("n_actions", I32), ("action", ActionDesc * MAX_ACTIONS),
                ("n_goal", I32), ("goal_obj", I32 * MAX_GOAL),
                ("lam", F * N_TERM_KINDS), ("eps", F * N_TERM_KINDS),
                ("lam_goal", F), ("lam_traj", F), ("eta", F),
                ("beta1", F), ("beta2", F), ("adam_eps", F),
                ("lr_conf", F), ("lr_pos", F), ("lr_yaw", F), ("lr_knot", F), ("grad_scale", F),
                ("lanes_per_particle", I32), ("block_threads", I32), ("block_sync", I32),
                ("self_collision", I32), ("collision_smooth", I32), ("ik_iters", I32), ("ik_damping", F), ("ik_seeds", I32)]


class Info(ctypes.Structure):
    _fields_ = [("D", I32), ("n_hard", I32), ("n_grasp", I32), ("n_fk", I32), ("term_kind", I32 * MAX_TERMS),
                ("n_local", I64), ("global_offset", I64), ("n_global", I64), ("t", I32),
                ("pairs_sphere_obb", I64), ("pairs_sphere_sphere", I64), ("n_kin", I32), ("n_place", I32),
                ("n_goal_pairs", I32), ("n_traj_seg", I32), ("n_robot_spheres", I32),
                ("lanes_per_particle", I32), ("block_threads", I32), ("block_sync", I32), ("pairs_self", I64),
                ("term_action", I32 * MAX_TERMS)]


EXPORTS = ["tamp_abi_version", "tamp_last_error", "tamp_sizeof_desc", "tamp_sizeof_info", "tamp_query_workspace",
           "tamp_init_problem", "tamp_get_info", "tamp_sample_particles", "tamp_optimize_step",
           "tamp_check_satisfied", "tamp_optimize_and_check", "tamp_best_k", "tamp_merge_best_k", "tamp_eval", "tamp_get_state",
           "tamp_set_state", "tamp_destroy", "tamp_kernel_launches", "tamp_plan_heuristic", "tamp_merge_scratch_bytes",
           "tamp_merge_records"]

_lib = None
_lib_path = None


def lib_path() -> str:
    """Path of the libtamp.so this process loaded (or would load)."""
    return _lib_path or LIB_PATH


def load(path: str = None):
    """Load the in-tree libtamp.so (raises if absent: the product path has no fallback).  `path` may name another
    in-tree build of the same library (A/B kernel experiments); it must live inside this repository."""
    global _lib, _lib_path
    if _lib is not None:
        return _lib
    path = os.path.abspath(path or LIB_PATH)
    root = os.path.dirname(HERE)
    if os.path.commonpath([path, root]) != root or os.path.basename(path) != "libtamp.so":
        raise RuntimeError(f"refusing to load {path}: only in-tree builds of libtamp.so")
    if not os.path.exists(path):
        raise RuntimeError(f"libtamp.so not built ({path}); run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    _lib_path = path
    vp, sz = ctypes.c_void_p, ctypes.c_size_t
    lib.tamp_abi_version.restype = I32
    lib.tamp_last_error.restype = ctypes.c_char_p
    lib.tamp_sizeof_desc.restype = sz
    lib.tamp_sizeof_info.restype = sz
    lib.tamp_query_workspace.argtypes = [vp, I64, ctypes.POINTER(sz)]
    lib.tamp_init_problem.argtypes = [vp, ctypes.c_int, I64, I64, I64, vp, sz, ctypes.POINTER(vp)]
    lib.tamp_get_info.argtypes = [vp, vp]
    lib.tamp_sample_particles.argtypes = [vp, ctypes.c_uint64, vp]
    lib.tamp_optimize_step.argtypes = [vp, I32, vp]
    lib.tamp_check_satisfied.argtypes = [vp, vp, vp, vp]
    lib.tamp_optimize_and_check.argtypes = [vp, I32, vp, vp, vp]
    lib.tamp_best_k.argtypes = [vp, I32, vp, vp]
    lib.tamp_merge_best_k.argtypes = [vp, vp, I32, I32, vp, vp]
    lib.tamp_eval.argtypes = [vp, vp, vp, vp, vp, vp]
    lib.tamp_get_state.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp]
    lib.tamp_set_state.argtypes = [vp, vp, vp, vp, vp, vp, I32, vp]
    lib.tamp_destroy.argtypes = [vp]
    lib.tamp_kernel_launches.restype = ctypes.c_uint64
    lib.tamp_plan_heuristic.restype = ctypes.c_double
    lib.tamp_plan_heuristic.argtypes = [vp, I32, ctypes.c_double]
    lib.tamp_merge_scratch_bytes.argtypes = [I32, ctypes.POINTER(sz)]
    lib.tamp_merge_scratch_bytes.restype = I32
    lib.tamp_merge_records.argtypes = [vp, I32, I32, I32, vp, vp, sz, vp]
    lib.tamp_merge_records.restype = I32
    for name in EXPORTS[4:15]:
        getattr(lib, name).restype = ctypes.c_int
    if lib.tamp_abi_version() != ABI_VERSION:
        raise RuntimeError("libtamp ABI version mismatch")
    if lib.tamp_sizeof_desc() != ctypes.sizeof(ProblemDesc) or lib.tamp_sizeof_info() != ctypes.sizeof(Info):
        raise RuntimeError("libtamp struct layout mismatch (rebuild)")
    _lib = lib
    return lib


class TampError(RuntimeError):
    pass


def _check(status: int):
    if status != 0:
        msg = _lib.tamp_last_error().decode()
        raise TampError(f"{STATUS.get(status, status)}: {msg}")


# ---------------------------------------------------------------------------------------------
# ProblemSpec (workloads/) -> tamp_problem_desc marshalling
# ---------------------------------------------------------------------------------------------
def _copy_floats(dst, values: np.ndarray):
    """Copy a contiguous float32 vector into the leading elements of a (nested) ctypes float array."""
    v = np.ascontiguousarray(values, dtype=np.float32)
    if v.nbytes > ctypes.sizeof(dst):
        raise ValueError("descriptor array too small")
    ctypes.memmove(ctypes.addressof(dst), v.ctypes.data, v.nbytes)


def build_desc(spec, grad_scale: float = 0.0, lanes_per_particle: int = 0, block_threads: int = 0,
               block_sync: int = -1) -> ProblemDesc:
    d = ProblemDesc()
    d.abi_version = ABI_VERSION
    r = spec.robot
    for j in range(NJ):
        for k in range(3):
            d.robot.dh[j][k] = float(r.dh[j][k])
        d.robot.joint_lo[j] = float(r.joint_lo[j])
        d.robot.joint_hi[j] = float(r.joint_hi[j])
    d.robot.flange_d, d.robot.tcp_yaw, d.robot.tcp_d = float(r.flange_d), float(r.tcp_yaw), float(r.tcp_d)
    for k in range(4):
        d.robot.base[k] = float(r.base[k])
    d.robot.n_spheres = len(r.spheres)
    _copy_floats(d.robot.sphere, np.asarray(r.spheres, dtype=np.float32).reshape(-1))
    for s in range(len(r.spheres)):
        d.robot.sphere_link[s] = int(r.sphere_link[s])
    masks = [0] * len(r.spheres)
    for i, j in getattr(r, "self_pairs", []):
        masks[i] |= 1 << j
        masks[j] |= 1 << i
    for i, m in enumerate(masks):
        d.robot.self_mask[i] = m
    d.n_obb = len(spec.obbs)
    for b, o in enumerate(spec.obbs):
        for k in range(3):
            d.obb[b].center[k] = float(o.center[k])
            d.obb[b].half[k] = float(o.half[k])
        d.obb[b].yaw = float(o.yaw)
        R = getattr(o, "R", None)
        if R is not None:                         # full orientation (box-to-world rotation, row-major)
            for k, v in enumerate(np.asarray(R, dtype=np.float32).reshape(9)):
                d.obb[b].rot[k] = float(v)
    d.n_objects = len(spec.objects)
    for i, o in enumerate(spec.objects):
        d.object[i].n_spheres = len(o.spheres)
        _copy_floats(d.object[i].sphere, np.asarray(o.spheres, dtype=np.float32).reshape(-1))
        d.object[i].footprint = float(o.footprint)
        d.object[i].grasp_xy = float(o.grasp_xy)
        d.object[i].grasp_z = float(o.grasp_z)
        d.object[i].grasp_mode = int(getattr(o, "grasp_mode", 0))
        d.object[i].grasp_y = float(getattr(o, "grasp_y", -1.0))
    d.n_surfaces = len(spec.surfaces)
    for i, s in enumerate(spec.surfaces):
        for k in range(4):
            d.surface[i].frame[k] = float(s.frame[k])
        for k in range(2):
            d.surface[i].lo[k] = float(s.lo[k])
            d.surface[i].hi[k] = float(s.hi[k])
        d.surface[i].support_obb = int(s.support_obb)
        d.surface[i].support_obj = int(s.support_obj)
    d.n_vars = len(spec.variables)
    for i, v in enumerate(spec.variables):
        dv = d.var[i]
        dv.kind, dv.is_const, dv.obj, dv.surface, dv.n_knots = int(v.kind), int(v.const), int(v.obj), int(v.surface), int(v.n_knots)
        if v.value is not None:
            for k in range(len(v.value)):
                dv.value[k] = float(v.value[k])
        dv.rng_stream = int(getattr(v, "rng_stream", 0)) & 0xFFFFFFFF
        for k in range(4):
            dv.lo[k] = float(v.lo[k]) if v.lo is not None else -math.inf
            dv.hi[k] = float(v.hi[k]) if v.hi is not None else math.inf
    d.n_actions = len(spec.actions)
    for i, a in enumerate(spec.actions):
        da = d.action[i]
        da.kind, da.obj, da.grasp, da.placement = int(a.kind), int(a.obj), int(a.grasp), int(a.placement)
        da.surface, da.q1, da.q2, da.traj = int(a.surface), int(a.q1), int(a.q2), int(a.traj)
    d.n_goal = len(spec.goal_objs)
    for i, o in enumerate(spec.goal_objs):
        d.goal_obj[i] = int(o)
    for k, name in enumerate(TERM_NAMES):
        d.lam[k] = float(spec.lam[name])
        d.eps[k] = float(spec.eps[name])
    d.lam_goal, d.lam_traj, d.eta = float(spec.lam_goal), float(spec.lam_traj), float(spec.eta)
    d.beta1, d.beta2, d.adam_eps = float(spec.beta1), float(spec.beta2), float(spec.adam_eps)
    d.lr_conf, d.lr_pos, d.lr_yaw, d.lr_knot = float(spec.lr_conf), float(spec.lr_pos), float(spec.lr_yaw), float(spec.lr_knot)
    d.grad_scale = float(grad_scale)
    d.lanes_per_particle = int(lanes_per_particle)
    d.block_threads = int(block_threads)
    d.block_sync = int(block_sync)
    d.self_collision = int(bool(getattr(spec, "self_collision", False)))
    d.collision_smooth = int(bool(getattr(spec, "collision_smooth", False)))
    d.ik_iters = int(getattr(spec, "ik_iters", 0))
    d.ik_damping = float(getattr(spec, "ik_damping", 0.1))
    d.ik_seeds = int(getattr(spec, "ik_seeds", 1))
    return d


def _ptr(t: Optional[torch.Tensor]):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream(device, stream=None):
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return ctypes.c_void_p(s.cuda_stream)


class TampContext:
    """One rank's particles of one skeleton on one GPU (tamp_ctx)."""

    def __init__(self, spec, n_local: int, global_offset: int = 0, n_global: Optional[int] = None,
                 device=None, grad_scale: float = 0.0, lanes_per_particle: int = 0, block_threads: int = 0,
                 block_sync: int = -1):
        self.lib = load()
        if not torch.cuda.is_available():
            raise RuntimeError("TampContext needs a CUDA device (no CPU fallback)")
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.n = int(n_local)
        self.gofs = int(global_offset)
        self.n_global = int(n_global if n_global is not None else n_local)
        self.desc = build_desc(spec, grad_scale, lanes_per_particle, block_threads, block_sync)
        nbytes = ctypes.c_size_t()
        _check(self.lib.tamp_query_workspace(ctypes.byref(self.desc), self.n, ctypes.byref(nbytes)))
        self.workspace = torch.empty(nbytes.value, dtype=torch.uint8, device=self.device)
        h = ctypes.c_void_p()
        _check(self.lib.tamp_init_problem(ctypes.byref(self.desc), self.device.index, self.n, self.gofs, self.n_global,
                                          _ptr(self.workspace), nbytes.value, ctypes.byref(h)))
        self.h = h
        info = Info()
        _check(self.lib.tamp_get_info(self.h, ctypes.byref(info)))
        self.D, self.n_hard, self.n_grasp, self.n_fk = info.D, info.n_hard, info.n_grasp, info.n_fk
        self.term_kinds = [TERM_NAMES[info.term_kind[i]] for i in range(self.n_hard)]
        self.term_actions = [int(info.term_action[i]) for i in range(self.n_hard)]
        self.work = dict(pairs_sphere_obb=info.pairs_sphere_obb, pairs_sphere_sphere=info.pairs_sphere_sphere,
                         n_kin=info.n_kin, n_place=info.n_place, n_goal_pairs=info.n_goal_pairs,
                         n_traj_seg=info.n_traj_seg, n_robot_spheres=info.n_robot_spheres, n_fk=info.n_fk,
                         D=info.D, pairs_self=info.pairs_self)
        self.lanes_per_particle = info.lanes_per_particle
        self.block_threads, self.block_sync = info.block_threads, info.block_sync
        self.counts_buf = torch.zeros(self.n_hard + 2, dtype=torch.int32, device=self.device)

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            self.lib.tamp_destroy(h)
            self.h = None

    @property
    def t(self) -> int:
        info = Info()
        _check(self.lib.tamp_get_info(self.h, ctypes.byref(info)))
        return info.t

    # ---- the five hot-path calls ----
    def sample(self, seed: int, stream=None):
        _check(self.lib.tamp_sample_particles(self.h, ctypes.c_uint64(seed), _stream(self.device, stream)))

    def optimize(self, n_steps: int, stream=None):
        _check(self.lib.tamp_optimize_step(self.h, int(n_steps), _stream(self.device, stream)))

    def check(self, cls: Optional[torch.Tensor] = None, counts: Optional[torch.Tensor] = None, stream=None):
        """Returns the counts tensor (device unless a host tensor is passed) and cls if given."""
        counts = self.counts_buf if counts is None else counts
        _check(self.lib.tamp_check_satisfied(self.h, _ptr(cls), _ptr(counts), _stream(self.device, stream)))
        return counts, cls

    def optimize_check(self, n_steps: int, cls: Optional[torch.Tensor] = None, counts: Optional[torch.Tensor] = None,
                       stream=None):
        """optimize(n_steps) then check(), one C-ABI call (the check rides on the last optimisation launch)."""
        counts = self.counts_buf if counts is None else counts
        _check(self.lib.tamp_optimize_and_check(self.h, int(n_steps), _ptr(cls), _ptr(counts),
                                                _stream(self.device, stream)))
        return counts, cls

    def best_k(self, k: int, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        out = torch.empty(k, self.D + 4, dtype=torch.float32, device=self.device) if out is None else out
        _check(self.lib.tamp_best_k(self.h, int(k), _ptr(out), _stream(self.device, stream)))
        return out

    def merge_best_k(self, records: torch.Tensor, k: int, stream=None) -> torch.Tensor:
        records = records.contiguous()
        out = torch.empty(k, self.D + 4, dtype=torch.float32, device=self.device)
        _check(self.lib.tamp_merge_best_k(self.h, _ptr(records), int(records.shape[0]), int(k), _ptr(out),
                                          _stream(self.device, stream)))
        return out

    # ---- inspection ----
    def eval(self, stream=None):
        J = torch.empty(self.n, dtype=torch.float32, device=self.device)
        soft = torch.empty_like(J)
        Jc = torch.empty(self.n, max(self.n_hard, 1), dtype=torch.float32, device=self.device)
        grad = torch.empty(self.n, self.D, dtype=torch.float32, device=self.device)
        _check(self.lib.tamp_eval(self.h, _ptr(J), _ptr(soft), _ptr(Jc), _ptr(grad), _stream(self.device, stream)))
        return J, soft, Jc[:, :self.n_hard], grad

    def get_state(self, stream=None):
        x = torch.empty(self.n, self.D, dtype=torch.float32, device=self.device)
        m, v = torch.empty_like(x), torch.empty_like(x)
        g = torch.empty(self.n, max(self.n_grasp, 1), 12, dtype=torch.float32, device=self.device)
        inv = torch.empty(self.n, dtype=torch.uint8, device=self.device)
        t = ctypes.c_int32()
        _check(self.lib.tamp_get_state(self.h, _ptr(x), _ptr(m), _ptr(v), _ptr(g), _ptr(inv), ctypes.byref(t),
                                       _stream(self.device, stream)))
        return dict(x=x, m=m, v=v, grasp=g[:, :self.n_grasp], invalid=inv, t=t.value)

    def set_state(self, x, grasp=None, m=None, v=None, invalid=None, t: int = 0, stream=None):
        def prep(a, dt):
            if a is None:
                return None
            a = torch.as_tensor(a, dtype=dt)
            return a.contiguous()
        x, m, v, grasp, invalid = (prep(x, torch.float32), prep(m, torch.float32), prep(v, torch.float32),
                                   prep(grasp, torch.float32), prep(invalid, torch.uint8))
        self._keep = (x, m, v, grasp, invalid)       # host tensors must outlive the async copy
        _check(self.lib.tamp_set_state(self.h, _ptr(x), _ptr(m), _ptr(v), _ptr(grasp), _ptr(invalid), int(t),
                                       _stream(self.device, stream)))


def merge_records(records: torch.Tensor, k: int, stream=None) -> torch.Tensor:
    """Stateless global top-k of best-k records [n][D+4] (tamp_merge_records; e.g. after an all-gather)."""
    lib = load()
    records = records.contiguous()
    n, width = int(records.shape[0]), int(records.shape[1])
    nb = ctypes.c_size_t()
    _check(lib.tamp_merge_scratch_bytes(n, ctypes.byref(nb)))
    scratch = torch.empty(nb.value + 256, dtype=torch.uint8, device=records.device)
    off = (-scratch.data_ptr()) % 256
    out = torch.empty(k, width, dtype=torch.float32, device=records.device)
    _check(lib.tamp_merge_records(_ptr(records), n, int(k), width - 4, _ptr(out),
                                  ctypes.c_void_p(scratch.data_ptr() + off), nb.value, _stream(records.device, stream)))
    return out


def plan_heuristic(counts, n_hard: int, penalty: float = -1e6) -> float:
    """Eq. 5 plan-feasibility heuristic from (all-reduced) satisfied counts (host)."""
    c = np.ascontiguousarray(np.asarray(counts if not torch.is_tensor(counts) else counts.cpu().numpy(), dtype=np.int32))
    return float(load().tamp_plan_heuristic(c.ctypes.data_as(ctypes.c_void_p), int(n_hard), float(penalty)))


def kernel_launches() -> int:
    """Kernels launched through libtamp by this process so far."""
    return int(load().tamp_kernel_launches())


def decode_records(rec: torch.Tensor):
    """Split best-k records [k][D+4] into (class int, cost float, global index int64, x [k][D])."""
    r = rec.detach().cpu().numpy()
    cls = r[:, 0].astype(np.int64)
    cost = r[:, 1].copy()
    lo = r[:, 2].copy().view(np.uint32).astype(np.int64)
    hi = r[:, 3].copy().view(np.int32).astype(np.int64)
    return cls, cost, lo | (hi << 32), r[:, 4:]
