"""Shared helpers for the GPU parity tests: identical seeded inputs for both sides, tolerances
(north_star: cost rel 1e-4, gradient rel 1e-3, 1-step state rel 1e-3; SURVEY §8(c) floors), and the
oracle-side kink detector used to exclude particles that sit on a non-differentiable point."""
import numpy as np
import torch

from oracle import tamp_oracle as O
from workloads import make_config

COST_RTOL, COST_ATOL = 1e-4, 1e-6
GRAD_RTOL = 1e-3
STEP_RTOL = 1e-3


def oracle_inputs(cfg, n, seed, gofs=0, self_collision=False):
    """Oracle-sampled particles rounded to fp32: the common starting state of both sides."""
    spec = make_config(cfg, n=n)
    spec.self_collision = self_collision
    csp = O.build_csp(spec)
    x, g = O.initialize_particles(spec, csp, seed, np.arange(gofs, gofs + n))
    x32, g32 = x.astype(np.float32), g.astype(np.float32)
    return spec, csp, x32, g32


def to_ctx_grasp(g32):
    n = g32.shape[0]
    return torch.from_numpy(np.ascontiguousarray(g32.reshape(n, -1, 12)))


def kink_mask(spec, csp, x64, g64, grad, rng, delta=1e-5, tries=2):
    """True where the oracle gradient jumps within +-delta of x along a random direction: the second
    difference g(x+d) - 2 g(x) + g(x-d) is O(delta^2) for a smooth cost but O(lambda) across a kink of a
    hinge / bound / box-SDF region switch (SURVEY §8(c) tolerance rules)."""
    bad = np.zeros(x64.shape[0], bool)
    scale = np.abs(grad).max(axis=1) + 1e-12
    for _ in range(tries):
        r = rng.normal(size=x64.shape)
        r /= np.linalg.norm(r, axis=1, keepdims=True)
        _, _, _, gp = O.cost_and_grad(spec, csp, x64 + delta * r, g64)
        _, _, _, gm = O.cost_and_grad(spec, csp, x64 - delta * r, g64)
        bad |= np.abs(gp - 2 * grad + gm).max(axis=1) > 0.1 * GRAD_RTOL * scale
    return bad


def grad_ok(g_gpu, g_or):
    err = np.abs(g_gpu - g_or).max(axis=1)
    return err <= GRAD_RTOL * np.abs(g_or).max(axis=1) + 1e-6
