"""Philox4x32-10 counter-based RNG (Salmon et al., SC'11 "Random123"), numpy uint64 arithmetic.

Used by the oracle's particle samplers.  The CUDA
path implements the same generator independently; only the algorithm is shared.

Counter convention for this project:
    key = (seed & 0xffffffff, seed >> 32)
    ctr = (global_particle_idx & 0xffffffff, global_particle_idx >> 32, variable_id, block)
    u_k = (word_k >> 8) * 2**-24          (k = 0..3, exact in float32)
"""
import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = np.uint64(0x9E3779B9)
W1 = np.uint64(0xBB67AE85)
MASK = np.uint64(0xFFFFFFFF)
S32 = np.uint64(32)


def philox4x32_10(ctr, key):
    """ctr: (..., 4) uint32-valued, key: (..., 2).  Returns (..., 4) uint32 words.

    One round: (hi0, lo0) = mulhilo(M0, c0); (hi1, lo1) = mulhilo(M1, c2);
    c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0); key bumped by (W0, W1) between rounds.
    """
    c = [np.asarray(ctr[..., i], dtype=np.uint64) & MASK for i in range(4)]
    k0 = np.asarray(key[..., 0], dtype=np.uint64) & MASK
    k1 = np.asarray(key[..., 1], dtype=np.uint64) & MASK
    for r in range(10):
        if r > 0:
            k0 = (k0 + W0) & MASK
            k1 = (k1 + W1) & MASK
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        hi0, lo0 = p0 >> S32, p0 & MASK
        hi1, lo1 = p1 >> S32, p1 & MASK
        c = [(hi1 ^ c[1] ^ k0) & MASK, lo1, (hi0 ^ c[3] ^ k1) & MASK, lo0]
    return np.stack(c, axis=-1).astype(np.uint32)


def uniforms(seed: int, gidx: np.ndarray, var_id: int, n: int) -> np.ndarray:
    """n uniforms in [0, 1) per particle for one variable: shape (len(gidx), n), float64 (exact fp32 values)."""
    gidx = np.asarray(gidx, dtype=np.uint64)
    nb = (n + 3) // 4
    out = np.empty((gidx.shape[0], nb * 4), dtype=np.float64)
    key = np.empty((gidx.shape[0], 2), dtype=np.uint64)
    key[:, 0] = np.uint64(seed & 0xFFFFFFFF)
    key[:, 1] = np.uint64((seed >> 32) & 0xFFFFFFFF)
    for b in range(nb):
        ctr = np.empty((gidx.shape[0], 4), dtype=np.uint64)
        ctr[:, 0] = gidx & MASK
        ctr[:, 1] = gidx >> S32
        ctr[:, 2] = np.uint64(var_id)
        ctr[:, 3] = np.uint64(b)
        w = philox4x32_10(ctr, key)
        out[:, 4 * b:4 * b + 4] = (w >> np.uint32(8)).astype(np.float64) * 2.0 ** -24
    return out[:, :n]
