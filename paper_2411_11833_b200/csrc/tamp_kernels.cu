// tamp_kernels.cu -- sm_100a kernels of the cuTAMP particle-optimisation hot path.
//
//   K1 k_sample      InitializeParticles: Philox4x32-10 counter RNG + samplers
//   K2 k_particle    fused Eq. 2 cost + hand-derived backward + Adam/projection, n_steps per launch
//                    (P:429-478); the same template also serves K3 (check, Eq. 3 + Eq. 5 counts) and
//                    the eval/inspection mode
//   K4 k_sort_chunk  best-k: bitonic sort of (key, payload) chunks, repeated until <= one chunk
//   K5 k_gather      records of the selected particles / merge of gathered records
//
// Mapping: one particle per 8-lane group, 4 particles per warp.  Lane l
// owns link frame l+1 of the 7-DOF chain (lane 7: the tool frame) and the <= 4 robot spheres on it.
// FK is an inclusive product scan of the per-joint transforms across the 8 lanes (3 shuffle steps);
// the backward is the reverse (suffix) scan of per-link wrenches:  dJ/dq_j = z_j . (M_j - o_j x F_j)
// with F_j, M_j the total force / moment (about the world origin) on links >= j.  Object spheres live
// in per-particle shared memory and are broadcast to the group; gradients on movable objects are
// accumulated as wrenches per object instance and converted to placement gradients at the end.
// No tensor cores: the math is 3x4 transform chains and pairwise distances (north_star).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <atomic>

#include "tamp_program.h"

namespace tamp {

constexpr unsigned FULL = 0xffffffffu;
constexpr float kPi = 3.14159265358979323846f;

// ------------------------------------------------------------------------------------------------
// small math
// ------------------------------------------------------------------------------------------------
struct M34 {
    float r[9];   // row-major rotation
    float t[3];
};

__device__ __forceinline__ M34 compose(const M34& a, const M34& b) {
    M34 c;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
#pragma unroll
        for (int j = 0; j < 3; ++j)
            c.r[3 * i + j] = fmaf(a.r[3 * i], b.r[j], fmaf(a.r[3 * i + 1], b.r[3 + j], a.r[3 * i + 2] * b.r[6 + j]));
        c.t[i] = fmaf(a.r[3 * i], b.t[0], fmaf(a.r[3 * i + 1], b.t[1], fmaf(a.r[3 * i + 2], b.t[2], a.t[i])));
    }
    return c;
}

__device__ __forceinline__ M34 shfl_m34(const M34& a, int src, int width = kGroup) {
    M34 o;
#pragma unroll
    for (int i = 0; i < 9; ++i) o.r[i] = __shfl_sync(FULL, a.r[i], src, width);
#pragma unroll
    for (int i = 0; i < 3; ++i) o.t[i] = __shfl_sync(FULL, a.t[i], src, width);
    return o;
}

__device__ __forceinline__ M34 shfl_up_m34(const M34& a, int d, int width = kGroup) {
    M34 o;
#pragma unroll
    for (int i = 0; i < 9; ++i) o.r[i] = __shfl_up_sync(FULL, a.r[i], d, width);
#pragma unroll
    for (int i = 0; i < 3; ++i) o.t[i] = __shfl_up_sync(FULL, a.t[i], d, width);
    return o;
}

__device__ __forceinline__ void load_m34(M34& a, const float* s) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        a.r[3 * i] = s[4 * i];
        a.r[3 * i + 1] = s[4 * i + 1];
        a.r[3 * i + 2] = s[4 * i + 2];
        a.t[i] = s[4 * i + 3];
    }
}

__device__ __forceinline__ void inv_m34(const M34& a, M34& o) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) o.r[3 * i + j] = a.r[3 * j + i];
#pragma unroll
    for (int i = 0; i < 3; ++i)
        o.t[i] = -(o.r[3 * i] * a.t[0] + o.r[3 * i + 1] * a.t[1] + o.r[3 * i + 2] * a.t[2]);
}

__device__ __forceinline__ void xform(const M34& T, float x, float y, float z, float& ox, float& oy, float& oz) {
    ox = fmaf(T.r[0], x, fmaf(T.r[1], y, fmaf(T.r[2], z, T.t[0])));
    oy = fmaf(T.r[3], x, fmaf(T.r[4], y, fmaf(T.r[5], z, T.t[1])));
    oz = fmaf(T.r[6], x, fmaf(T.r[7], y, fmaf(T.r[8], z, T.t[2])));
}

template <int GS>
__device__ __forceinline__ float gsum(float v) {      // butterfly sum over the GS lanes of a particle group
#pragma unroll
    for (int m = 1; m < GS; m <<= 1) v += __shfl_xor_sync(FULL, v, m);
    return v;
}

// sin/cos without the large-argument (Payne-Hanek) path of sincosf: Cody-Waite reduction by pi/2 with a
// three-part constant (exact for |x| < ~1e4; joint angles and yaws are within a few radians) and the
// cephes single-precision minimax polynomials on [-pi/4, pi/4] (<= 2 ulp).  Branch-free and compact, so
// the step loop's instruction footprint stays small.
__device__ __forceinline__ void fsincos(float x, float* s, float* c) {
    const float k = rintf(x * 0.636619772367581343f);
    float r = fmaf(k, -1.57079601287841796875f, x);
    r = fmaf(k, -3.13916473e-07f, r);
    r = fmaf(k, -5.39030253e-15f, r);
    const float r2 = r * r;
    const float ps = fmaf(fmaf(fmaf(-1.9515295891e-4f, r2, 8.3321608736e-3f), r2, -1.6666654611e-1f), r2 * r, r);
    const float pc = fmaf(fmaf(fmaf(fmaf(2.443315711809948e-5f, r2, -1.388731625493765e-3f), r2,
                                    4.166664568298827e-2f), r2, -0.5f), r2, 1.0f);
    const int q = (int)k;
    const float sv = (q & 1) ? pc : ps;
    const float cv = (q & 1) ? ps : pc;
    *s = (q & 2) ? -sv : sv;
    *c = ((q + 1) & 2) ? -cv : cv;
}

// atan2(y, x) for y >= 0 (an angle in [0, pi]): octant reduction, cephes atanf reduction at tan(pi/8) and its
// single-precision polynomial (max |err| 2.7e-7 rad over [0, pi], ~1 ulp; verified on the host against
// libm atan2); branch-free and shorter than atan2f
__device__ __forceinline__ float fatan2_pos(float y, float x) {
    const float ax = fabsf(x);
    const float mx = fmaxf(ax, y), mn = fminf(ax, y);
    const float a = mx > 0.f ? mn / mx : 0.f;
    const bool big = a > 0.41421356f;
    const float t = big ? (a - 1.f) / (a + 1.f) : a;
    const float z = t * t;
    const float p = fmaf(fmaf(fmaf(8.05374449538e-2f, z, -1.38776856032e-1f), z, 1.99777106478e-1f), z, -3.33329491539e-1f);
    float r = fmaf(p * z, t, t) + (big ? 0.785398163397f : 0.f);
    r = y > ax ? 1.57079632679f - r : r;
    return x < 0.f ? 3.14159265359f - r : r;
}

struct Wrench {
    float f[3];
    float m[3];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i < 3; ++i) f[i] = m[i] = 0.f;
    }
    // force g applied at point w: F += g, M += w x g
    __device__ __forceinline__ void add_point(float wx, float wy, float wz, float gx, float gy, float gz) {
        f[0] += gx; f[1] += gy; f[2] += gz;
        m[0] = fmaf(wy, gz, fmaf(-wz, gy, m[0]));
        m[1] = fmaf(wz, gx, fmaf(-wx, gz, m[1]));
        m[2] = fmaf(wx, gy, fmaf(-wy, gx, m[2]));
    }
    __device__ __forceinline__ bool nonzero() const {
        return (f[0] != 0.f) | (f[1] != 0.f) | (f[2] != 0.f) | (m[0] != 0.f) | (m[1] != 0.f) | (m[2] != 0.f);
    }
    template <int GS>
    __device__ __forceinline__ void group_sum() {
#pragma unroll
        for (int i = 0; i < 3; ++i) { f[i] = gsum<GS>(f[i]); m[i] = gsum<GS>(m[i]); }
    }
};

// ------------------------------------------------------------------------------------------------
// collision primitives (hinge max(0, r + eta - sd), L1)
// ------------------------------------------------------------------------------------------------
// Sphere vs OBB.  Returns the hinge value; if GRAD adds lam * dJ/dw to (gx, gy, gz).
template <bool GRAD>
__device__ __forceinline__ float sphere_obb(float wx, float wy, float wz, float rr, const KObb& B, float lam,
                                            float& gx, float& gy, float& gz) {
    const float dx = wx - B.c[0], dy = wy - B.c[1], dz = wz - B.c[2];
    const float px = fmaf(B.R[0], dx, fmaf(B.R[3], dy, B.R[6] * dz));
    const float py = fmaf(B.R[1], dx, fmaf(B.R[4], dy, B.R[7] * dz));
    const float pz = fmaf(B.R[2], dx, fmaf(B.R[5], dy, B.R[8] * dz));
    const float ax = fabsf(px) - B.h[0], ay = fabsf(py) - B.h[1], az = fabsf(pz) - B.h[2];
    const float qx = fmaxf(ax, 0.f), qy = fmaxf(ay, 0.f), qz = fmaxf(az, 0.f);
    const float s = fmaf(qx, qx, fmaf(qy, qy, qz * qz));
    const float mx = fmaxf(ax, fmaxf(ay, az));
    if (mx > 0.f && s >= rr * rr) return 0.f;          // outside and beyond reach: inactive
    float sd, gpx, gpy, gpz;
    if (s > 1e-30f) {                                    // outside: sd = ||max(a, 0)||
        const float inv = rsqrtf(s);
        sd = s * inv;
        gpx = copysignf(qx * inv, px);
        gpy = copysignf(qy * inv, py);
        gpz = copysignf(qz * inv, pz);
    } else {                                             // inside: sd = max_k a_k, grad sign(p_k) e_k
        sd = mx;
        int k = 0;
        float best = ax;
        if (ay > best) { k = 1; best = ay; }
        if (az > best) { k = 2; }
        gpx = (k == 0) ? copysignf(1.f, px) : 0.f;
        gpy = (k == 1) ? copysignf(1.f, py) : 0.f;
        gpz = (k == 2) ? copysignf(1.f, pz) : 0.f;
    }
    const float pen = rr - sd;
    if (!(pen > 0.f)) return 0.f;
    if (GRAD) {   // dJ/dw = -R grad_p
        gx = fmaf(-lam, fmaf(B.R[0], gpx, fmaf(B.R[1], gpy, B.R[2] * gpz)), gx);
        gy = fmaf(-lam, fmaf(B.R[3], gpx, fmaf(B.R[4], gpy, B.R[5] * gpz)), gy);
        gz = fmaf(-lam, fmaf(B.R[6], gpx, fmaf(B.R[7], gpy, B.R[8] * gpz)), gz);
    }
    return pen;
}

// Sphere vs sphere.  Returns the hinge; if GRAD: (ux, uy, uz) = lam * (w_a - w_b)/||.|| (0 if inactive).
template <bool GRAD>
__device__ __forceinline__ float sphere_sphere(float ax, float ay, float az, float rr, float4 b,
                                               float lam, float& ux, float& uy, float& uz) {
    const float dx = ax - b.x, dy = ay - b.y, dz = az - b.z;
    const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    const float R = rr + b.w;
    ux = uy = uz = 0.f;
    if (fmaf(-R, R, d2) >= 0.f) return 0.f;
    if (d2 > 0.f) {
        const float inv = rsqrtf(d2);
        const float pen = R - d2 * inv;
        if (!(pen > 0.f)) return 0.f;
        if (GRAD) {
            const float k = lam * inv;
            ux = dx * k; uy = dy * k; uz = dz * k;
        }
        return pen;
    }
    return R;   // coincident centres: cost R, zero gradient (L13)
}

constexpr float kFar = 1e18f;   // position of padded (absent) spheres: never within reach of anything

// NS query spheres per lane (registers) vs the 8 (padded) spheres of one object instance (shared memory,
// broadcast to the group).  Fast path: branch-free test of all NS x 8 pairs (d^2 - (ra+rb)^2 < 0 ?), no
// square roots; only if some pair of the warp is active are the hinges and gradients evaluated.
// Returns the hinge sum; if GRAD accumulates dJ/dw_a (x lam) into g and the partner's wrench into pw.
template <bool GRAD, int NS, class OnWrench>
__device__ __forceinline__ float pairs_vs_instance(const float (&w)[NS][3], const float (&rr)[NS], const float4* Bs,
                                                   const float4 bound, float lam, float (&g)[NS][3], OnWrench&& on_wrench) {
    // broad phase: skip the instance unless some query sphere of the warp reaches its bounding sphere
    float mb = 1.f;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        const float dx = w[k][0] - bound.x, dy = w[k][1] - bound.y, dz = w[k][2] - bound.z;
        const float R = rr[k] + bound.w;
        mb = fminf(mb, fmaf(-R, R, fmaf(dx, dx, fmaf(dy, dy, dz * dz))));
    }
    if (!__any_sync(FULL, mb < 0.f)) return 0.f;
    // narrow phase, branch-free: which of the NS x 8 pairs reach (d^2 < (ra + rb)^2)?
    uint32_t act[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) act[k] = 0u;
#pragma unroll
    for (int b = 0; b < TAMP_MAX_OBJ_SPHERES; ++b) {
        const float4 B = Bs[b];
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            const float dx = w[k][0] - B.x, dy = w[k][1] - B.y, dz = w[k][2] - B.z;
            const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
            const float R = rr[k] + B.w;
            act[k] |= (fmaf(-R, R, d2) < 0.f ? 1u : 0u) << b;
        }
    }
    uint32_t any = 0u;
#pragma unroll
    for (int k = 0; k < NS; ++k) any |= act[k];
    float j = 0.f;
    if (__any_sync(FULL, any != 0u)) {
        // hinges and gradients of the active pairs only
        Wrench pw;
        pw.zero();
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            uint32_t m = act[k];
            while (m) {
                const int b = __ffs(m) - 1;
                m &= m - 1u;
                const float4 B = Bs[b];
                float ux, uy, uz;
                j += sphere_sphere<GRAD>(w[k][0], w[k][1], w[k][2], rr[k], B, lam, ux, uy, uz);
                if (GRAD) {
                    g[k][0] -= ux; g[k][1] -= uy; g[k][2] -= uz;
                    pw.add_point(B.x, B.y, B.z, ux, uy, uz);
                }
            }
        }
        on_wrench(pw);   // warp-uniform: reduce / store the partner's wrench
    }
    return j;
}

// NS query spheres per lane vs one OBB: branch-free reject (outside and |max(a,0)|^2 >= r^2), exact
// hinge + gradient only if some sphere of the warp reaches the box.
template <bool GRAD, int NS>
__device__ __forceinline__ float spheres_vs_obb(const float (&w)[NS][3], const float (&rr)[NS], const KObb& B,
                                                float lam, float (&g)[NS][3]) {
    // broad phase: bounding sphere of the box
    float mb = 1.f;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        const float dx = w[k][0] - B.c[0], dy = w[k][1] - B.c[1], dz = w[k][2] - B.c[2];
        const float R = rr[k] + B.rad;
        mb = fminf(mb, fmaf(-R, R, fmaf(dx, dx, fmaf(dy, dy, dz * dz))));
    }
    if (!__any_sync(FULL, mb < 0.f)) return 0.f;
    float mn = 1.f;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        const float dx = w[k][0] - B.c[0], dy = w[k][1] - B.c[1], dz = w[k][2] - B.c[2];
        const float px = fmaf(B.R[0], dx, fmaf(B.R[3], dy, B.R[6] * dz));
        const float py = fmaf(B.R[1], dx, fmaf(B.R[4], dy, B.R[7] * dz));
        const float pz = fmaf(B.R[2], dx, fmaf(B.R[5], dy, B.R[8] * dz));
        const float ax = fabsf(px) - B.h[0], ay = fabsf(py) - B.h[1], az = fabsf(pz) - B.h[2];
        const float qx = fmaxf(ax, 0.f), qy = fmaxf(ay, 0.f), qz = fmaxf(az, 0.f);
        const float s = fmaf(qx, qx, fmaf(qy, qy, qz * qz));
        const float mx = fmaxf(ax, fmaxf(ay, az));
        mn = fminf(mn, mx > 0.f ? fmaf(-rr[k], rr[k], s) : -1.f);
    }
    float j = 0.f;
    if (__any_sync(FULL, mn < 0.f)) {
#pragma unroll
        for (int k = 0; k < NS; ++k) j += sphere_obb<GRAD>(w[k][0], w[k][1], w[k][2], rr[k], B, lam, g[k][0], g[k][1], g[k][2]);
    }
    return j;
}

__device__ __forceinline__ void add_wrench(float* dst, const Wrench& w) {
    dst[0] += w.f[0]; dst[1] += w.f[1]; dst[2] += w.f[2];
    dst[3] += w.m[0]; dst[4] += w.m[1]; dst[5] += w.m[2];
}

// reduce a per-lane partner wrench over the group and add it to the instance accumulator (lane 0)
template <bool GRAD, int GS>
__device__ __forceinline__ void flush_partner(Wrench& pw, bool movable, float* dst, int gl) {
    if (GRAD && movable && __any_sync(FULL, pw.nonzero())) {
        pw.template group_sum<GS>();
        if (gl == 0) add_wrench(dst, pw);
    }
}

// phase-B variant: each 8-lane half may work on a different FK instance (so `movable` and `dst` may differ
// between halves): warp-uniform vote, per-half reduction, halves add one after the other (deterministic).
template <bool GRAD, int HP, int LPF>
__device__ __forceinline__ void flush_partner_b(Wrench& pw, bool movable, float* dst, int ll, int half, bool real) {
    if (!GRAD) return;
    if (__any_sync(FULL, movable && pw.nonzero())) {
        pw.template group_sum<LPF>();
#pragma unroll
        for (int h = 0; h < HP; ++h) {
            if (half == h && ll == 0 && real && movable) add_wrench(dst, pw);
            if (HP > 1) __syncwarp();
        }
    }
}

// ------------------------------------------------------------------------------------------------
// K2 / K3 / eval: the fused per-particle kernel
// ------------------------------------------------------------------------------------------------
template <int MODE>
struct TermSink {
    float J = 0.f;
    bool sat = true;
};

template <int MODE>
__device__ __forceinline__ void finish_term(const KProgram& P, const KArgs& A, TermSink<MODE>& sink, int term,
                                            float val, int gl, bool active, int64_t p, int* s_counts,
                                            bool real = true) {
    if (!real) return;   // ghost FK instance (pair padding)
    sink.J = fmaf(P.term_lam[term], val, sink.J);
    if (MODE == MODE_EVAL) {
        if (gl == 0 && active && A.out_Jc) A.out_Jc[p * P.n_terms + term] = val;
    } else if (MODE == MODE_CHECK) {
        const bool ok = val <= P.term_eps[term];
        sink.sat = sink.sat && ok;
        if (gl == 0 && active && ok) atomicAdd(&s_counts[term], 1);
    }
}

// Particle-group mapping.  LPF = lanes per FK instance: 8 (lane l owns link frame l+1; lane 7 the tool
// frame) or 4 (lane l owns link frames 2l+1 and 2l+2: half the warp-instructions per particle for the
// per-particle serial work -- FK scan, Kin, bookkeeping -- twice the sphere work per lane).  HP = FK
// instances a particle group processes concurrently: 1, or 2 (two LPF-lane halves run the two FK instances
// of a pair of identical structure).  GS = LPF * HP lanes per particle.
// BSYNC: block-synchronous phases so that all warps of a block execute the same code region at a time and
// share the instruction cache.  0 = off (warp-level only), 1 = at phase boundaries, 2 = also after every
// FK instance.
template <int MODE, int LPF, int HP, int BSYNC>
__global__ void __launch_bounds__(LPF == 4 ? 512 : 768, 1) k_particle(const __grid_constant__ KProgram P, const KArgs A) {
    constexpr bool GRAD = MODE != MODE_CHECK;
    constexpr int GS = LPF * HP;                                   // lanes per particle
    constexpr int LPL = kGroup / LPF;                              // link frames per lane
    constexpr int NS = TAMP_MAX_SPHERES_PER_LINK * LPL;            // robot spheres per lane
    constexpr int NH = TAMP_MAX_OBJ_SPHERES / LPF;                 // held-object spheres per lane
    constexpr int NSO = GS >= TAMP_MAX_OBJ_SPHERES ? 1 : TAMP_MAX_OBJ_SPHERES / GS;   // placed-object spheres per lane
    constexpr int NJL = (TAMP_NJ + GS - 1) / GS;                   // joints per lane in trajectory costs
    extern __shared__ float4 smem4[];
    __shared__ float4 s_osph[TAMP_MAX_OBJECTS][TAMP_MAX_OBJ_SPHERES];
    __shared__ int s_counts[TAMP_MAX_TERMS + 2];
    __shared__ float4 s_F[kGroup][3];                              // fixed transform of each joint (7: tool)
    __shared__ float4 s_rsph[kGroup][TAMP_MAX_SPHERES_PER_LINK];   // spheres of each link frame
    __shared__ uint32_t s_selfmask[kGroup * TAMP_MAX_SPHERES_PER_LINK];

    const int gl = threadIdx.x & (GS - 1);          // lane within the particle group
    const int ll = gl & (LPF - 1);                  // lane within the FK segment
    const int half = gl / LPF;                      // HP = 2: which FK instance of the pair
    const int grp = threadIdx.x / GS;
    const int64_t pid = (int64_t)blockIdx.x * (blockDim.x / GS) + grp;
    const bool active = pid < A.n;
    const int64_t p = active ? pid : (A.n - 1);
    float* S = reinterpret_cast<float*>(smem4) + (size_t)grp * A.stride;
    float* xs = S;
    float* gs = S + A.off_g;
    float* ipose = S + A.off_ipose;
    float4* isph = reinterpret_cast<float4*>(S + A.off_isph);
    float* iwr = S + A.off_iwr;
    float* gT = S + A.off_gT;
    float* gTi = S + A.off_gTi;
    const int D = P.D;
    auto phase_sync = [&]() {
        if (BSYNC > 0) __syncthreads(); else __syncwarp();
    };
    auto ibound = [&](int i) { return *reinterpret_cast<const float4*>(ipose + 16 * i + 12); };

    for (int i = threadIdx.x; i < TAMP_MAX_OBJECTS * TAMP_MAX_OBJ_SPHERES; i += blockDim.x) {
        const int o = i / TAMP_MAX_OBJ_SPHERES, k = i % TAMP_MAX_OBJ_SPHERES;
        s_osph[o][k] = make_float4(P.osph[o][k][0], P.osph[o][k][1], P.osph[o][k][2], P.osph[o][k][3]);
    }
    if (MODE == MODE_CHECK)
        for (int i = threadIdx.x; i < P.n_terms + 2; i += blockDim.x) s_counts[i] = 0;
    if (threadIdx.x < kGroup * 3) {
        const int l = threadIdx.x / 3, r = threadIdx.x % 3;
        s_F[l][r] = make_float4(P.F[l][4 * r], P.F[l][4 * r + 1], P.F[l][4 * r + 2], P.F[l][4 * r + 3]);
    }
    if (threadIdx.x < kGroup * TAMP_MAX_SPHERES_PER_LINK) {
        const int l = threadIdx.x / TAMP_MAX_SPHERES_PER_LINK, k = threadIdx.x % TAMP_MAX_SPHERES_PER_LINK;
        s_rsph[l][k] = make_float4(P.rsph[l][k][0], P.rsph[l][k][1], P.rsph[l][k][2], P.rsph[l][k][3]);
        s_selfmask[threadIdx.x] = P.self_mask[threadIdx.x];
    }
    float4* rsw = reinterpret_cast<float4*>(S + A.off_rsw) + (HP > 1 ? half : 0) * (kGroup * TAMP_MAX_SPHERES_PER_LINK + kGroup);
    float4* rlb = rsw + kGroup * TAMP_MAX_SPHERES_PER_LINK;       // world bounding sphere of each link frame
    int nsph[LPL];
    float jlo[LPL], jhi[LPL];
#pragma unroll
    for (int u = 0; u < LPL; ++u) {
        const int j = ll * LPL + u;                  // joint j+1 / link frame j+1 (j = 7: tool)
        nsph[u] = P.rsph_n[j];
        jlo[u] = j < TAMP_NJ ? P.jlo[j] : 0.f;
        jhi[u] = j < TAMP_NJ ? P.jhi[j] : 0.f;
    }

    // particle state -> shared memory
    const float* xg = A.x + p * D;
    for (int d = gl; d < D; d += GS) xs[d] = xg[d];
    for (int i = gl; i < P.n_grasp * 12; i += GS) gT[(i / 12) * 16 + (i % 12)] = A.grasp[(p * P.n_grasp) * 12 + i];
    bool invalid = A.invalid[p] != 0;
    __syncthreads();
    if (gl == 0) {
        for (int k = 0; k < P.n_grasp; ++k) {
            M34 g, gi;
            load_m34(g, gT + 16 * k);
            inv_m34(g, gi);
            float* o = gTi + 16 * k;
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                o[4 * i] = gi.r[3 * i]; o[4 * i + 1] = gi.r[3 * i + 1]; o[4 * i + 2] = gi.r[3 * i + 2];
                o[4 * i + 3] = gi.t[i];
            }
        }
    }
    __syncwarp();

    const int n_iter = (MODE == MODE_OPT) ? A.n_steps : 1;
    for (int it = 0; it < n_iter; ++it) {
        TermSink<MODE> sink;
        float soft = 0.f;

        // ---- phase A: object instances (poses, world sphere centres), zero accumulators ----
        for (int i = 0; i < P.n_inst; ++i) {
            const KInst& I = P.inst[i];
            if (I.xoff < 0 && it > 0) continue;      // constant instances: set up once per launch
            float px, py, pz, yaw;
            if (I.xoff >= 0) { px = xs[I.xoff]; py = xs[I.xoff + 1]; pz = xs[I.xoff + 2]; yaw = xs[I.xoff + 3]; }
            else { px = I.pose[0]; py = I.pose[1]; pz = I.pose[2]; yaw = I.pose[3]; }
            float sy, cy;
            fsincos(yaw, &sy, &cy);
            float* ip = ipose + 16 * i;      // [R row0 | t0, R row1 | t1, R row2 | t2, bounding sphere]
            if (gl == 0) {
                ip[0] = cy; ip[1] = -sy; ip[2] = 0.f; ip[3] = px;
                ip[4] = sy; ip[5] = cy; ip[6] = 0.f; ip[7] = py;
                ip[8] = 0.f; ip[9] = 0.f; ip[10] = 1.f; ip[11] = pz;
                const float* ob = P.obound[I.obj];   // world bounding sphere (broad phase)
                ip[12] = fmaf(cy, ob[0], fmaf(-sy, ob[1], px));
                ip[13] = fmaf(sy, ob[0], fmaf(cy, ob[1], py));
                ip[14] = pz + ob[2];
                ip[15] = ob[3];
            }
            for (int k = gl; k < TAMP_MAX_OBJ_SPHERES; k += GS) {
                const float4 c = s_osph[I.obj][k];
                isph[i * TAMP_MAX_OBJ_SPHERES + k] = k < P.osph_n[I.obj]
                    ? make_float4(fmaf(cy, c.x, fmaf(-sy, c.y, px)), fmaf(sy, c.x, fmaf(cy, c.y, py)), pz + c.z, c.w)
                    : make_float4(kFar, kFar, kFar, 0.f);
            }
            if (GRAD)
                for (int c = gl; c < 6; c += GS) iwr[8 * i + c] = 0.f;
        }
        if (GRAD) for (int d = gl; d < D; d += GS) gs[d] = 0.f;
        phase_sync();

        // ---- phase B: robot configurations (Pick/Place confs, knots) ----
        // HP = 2: the two halves process the two FK instances of a pair of identical structure concurrently
        // (the compiler pairs them; an unmatched instance is paired with a ghost copy whose results are
        // discarded), so control flow stays warp-uniform.  HP = 1: ghosts are skipped.
        TermSink<MODE> sinkB;                  // this half's share of the phase-B terms
        for (int f0 = 0; f0 < P.n_fk; f0 += HP) {
            const KFk K = P.fk[f0 + (HP > 1 ? half : 0)];
            const bool real = !K.ghost;
            if (HP == 1 && !real) continue;
            // A_j = F_j Rz(q_j) for my joints, local product, product scan over the LPF lanes (FK)
            float q[LPL];
            M34 Al[LPL];
#pragma unroll
            for (int u = 0; u < LPL; ++u) {
                const int j = ll * LPL + u;
                q[u] = j < TAMP_NJ ? xs[K.xoff + j] : 0.f;
                float s, c;
                fsincos(q[u], &s, &c);
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    const float4 f4 = s_F[j][i];
                    Al[u].r[3 * i] = fmaf(f4.x, c, f4.y * s);
                    Al[u].r[3 * i + 1] = fmaf(f4.y, c, -f4.x * s);
                    Al[u].r[3 * i + 2] = f4.z;
                    Al[u].t[i] = f4.w;
                }
            }
            M34 Sc = Al[0];
            if (LPL == 2) Sc = compose(Al[0], Al[LPL - 1]);
#pragma unroll
            for (int d = 1; d < LPF; d <<= 1) {
                const M34 U = shfl_up_m34(Sc, d, LPF);
                if (ll >= d) Sc = compose(U, Sc);
            }
            M34 T[LPL];                       // my link frames (world)
            if (LPL == 1) {
                T[0] = Sc;
            } else {
                const M34 E = shfl_up_m34(Sc, 1, LPF);     // product of all earlier lanes' transforms
                T[0] = ll == 0 ? Al[0] : compose(E, Al[0]);
                T[LPL - 1] = Sc;
            }
            const float lam_cf = K.term_cf >= 0 ? P.term_lam[K.term_cf] : 0.f;
            // my links' spheres in the world
            float w[NS][3], gw[NS][3], rr[NS];
#pragma unroll
            for (int u = 0; u < LPL; ++u)
#pragma unroll
                for (int k = 0; k < TAMP_MAX_SPHERES_PER_LINK; ++k) {
                    const int s = u * TAMP_MAX_SPHERES_PER_LINK + k;
                    const float4 c4 = s_rsph[ll * LPL + u][k];
                    xform(T[u], c4.x, c4.y, c4.z, w[s][0], w[s][1], w[s][2]);
                    if (k >= nsph[u]) w[s][0] = w[s][1] = w[s][2] = kFar;      // absent sphere slot
                    rr[s] = c4.w + P.eta;
                    gw[s][0] = gw[s][1] = gw[s][2] = 0.f;
                }
            float jcf = 0.f;
            if (K.term_cf >= 0) {
                // robot spheres vs OBBs (constant cache)
                for (int b = 0; b < P.n_obb; ++b)
                    if ((K.obb_mask >> b) & 1) jcf += spheres_vs_obb<GRAD, NS>(w, rr, P.obb[b], lam_cf, gw);
                // robot spheres vs movable objects' spheres (shared memory)
                for (int pi = 0; pi < K.part_count; ++pi) {
                    const int ii = P.partners[K.part_begin + pi];
                    jcf += pairs_vs_instance<GRAD, NS>(w, rr, isph + ii * TAMP_MAX_OBJ_SPHERES, ibound(ii), lam_cf, gw,
                        [&](Wrench& pw) { flush_partner_b<GRAD, HP, LPF>(pw, P.inst[ii].xoff >= 0, iwr + 8 * ii, ll, half, real); });
                }
            }
            // robot self-collision: every lane tests its own spheres against their pair
            // partners (sphere centres shared through shared memory), keeping only its own spheres' gradient;
            // each pair's hinge is counted once, by the lower sphere id.
            if (K.term_self >= 0) {
#pragma unroll
                for (int s = 0; s < NS; ++s)
                    rsw[ll * NS + s] = make_float4(w[s][0], w[s][1], w[s][2], rr[s] - P.eta);
#pragma unroll
                for (int u = 0; u < LPL; ++u) {
                    const float* lb = P.lbound[ll * LPL + u];
                    float bx, by, bz;
                    xform(T[u], lb[0], lb[1], lb[2], bx, by, bz);
                    rlb[ll * LPL + u] = make_float4(bx, by, bz, lb[3] + P.eta);
                }
                __syncwarp();
                float js = 0.f;
                const float lam_self = P.term_lam[K.term_self];
#pragma unroll
                for (int u = 0; u < LPL; ++u) {
                    // broad phase: links whose bounding spheres overlap this link's
                    const float4 a4 = rlb[ll * LPL + u];
                    uint32_t near = 0u;
#pragma unroll
                    for (int m = 0; m < kGroup; ++m) {
                        const float4 b4 = rlb[m];
                        const float dx = a4.x - b4.x, dy = a4.y - b4.y, dz = a4.z - b4.z;
                        const float R = a4.w + b4.w;
                        near |= (fmaf(-R, R, fmaf(dx, dx, fmaf(dy, dy, dz * dz))) < 0.f ? 0xFu : 0u) << (4 * m);
                    }
#pragma unroll
                    for (int k = 0; k < TAMP_MAX_SPHERES_PER_LINK; ++k) {
                        const int s = u * TAMP_MAX_SPHERES_PER_LINK + k;
                        const int sid = ll * NS + s;
                        uint32_t m = s_selfmask[sid] & near;
                        while (m) {
                            const int t = __ffs(m) - 1;
                            m &= m - 1u;
                            float ux, uy, uz;
                            const float pen = sphere_sphere<GRAD>(w[s][0], w[s][1], w[s][2], rr[s], rsw[t], lam_self, ux, uy, uz);
                            if (sid < t) js += pen;
                            if (GRAD) { gw[s][0] -= ux; gw[s][1] -= uy; gw[s][2] -= uz; }
                        }
                    }
                }
                finish_term<MODE>(P, A, sinkB, K.term_self, gsum<LPF>(js), ll, active, p, s_counts, real);
                __syncwarp();
            }
            Wrench Wl[LPL];                   // wrench (about the world origin) on each of my links
#pragma unroll
            for (int u = 0; u < LPL; ++u) {
                Wl[u].zero();
                if (GRAD) {
#pragma unroll
                    for (int k = 0; k < TAMP_MAX_SPHERES_PER_LINK; ++k) {
                        const int s = u * TAMP_MAX_SPHERES_PER_LINK + k;
                        Wl[u].add_point(w[s][0], w[s][1], w[s][2], gw[s][0], gw[s][1], gw[s][2]);
                    }
                }
            }
            // tool frame to every lane of the segment
            const M34 Tee = shfl_m34(T[LPL - 1], LPF - 1, LPF);
            // held object at a MoveHold knot: attached spheres T_ee T(g)^-1 c (CFreeTrajHold)
            if (K.held_grasp >= 0 && K.term_cf >= 0) {
                M34 Gi, Tobj;
                load_m34(Gi, gTi + 16 * K.held_grasp);
                Tobj = compose(Tee, Gi);
                const int ho = K.held_obj;
                float h[NH][3], gh[NH][3], hr[NH];
#pragma unroll
                for (int v = 0; v < NH; ++v) {
                    const int k = ll + LPF * v;
                    const float4 c = s_osph[ho][k];
                    xform(Tobj, c.x, c.y, c.z, h[v][0], h[v][1], h[v][2]);
                    if (k >= P.osph_n[ho]) h[v][0] = h[v][1] = h[v][2] = kFar;
                    hr[v] = c.w + P.eta;
                    gh[v][0] = gh[v][1] = gh[v][2] = 0.f;
                }
                for (int b = 0; b < P.n_obb; ++b)
                    if ((K.obb_mask >> b) & 1) jcf += spheres_vs_obb<GRAD, NH>(h, hr, P.obb[b], lam_cf, gh);
                for (int pi = 0; pi < K.part_count; ++pi) {
                    const int ii = P.partners[K.part_begin + pi];
                    jcf += pairs_vs_instance<GRAD, NH>(h, hr, isph + ii * TAMP_MAX_OBJ_SPHERES, ibound(ii), lam_cf, gh,
                        [&](Wrench& pw) { flush_partner_b<GRAD, HP, LPF>(pw, P.inst[ii].xoff >= 0, iwr + 8 * ii, ll, half, real); });
                }
                if (GRAD) {   // held-object wrench acts on the tool link (last lane of the segment)
                    Wrench hw;
                    hw.zero();
#pragma unroll
                    for (int v = 0; v < NH; ++v) hw.add_point(h[v][0], h[v][1], h[v][2], gh[v][0], gh[v][1], gh[v][2]);
                    hw.template group_sum<LPF>();
                    if (ll == LPF - 1) {
#pragma unroll
                        for (int i = 0; i < 3; ++i) { Wl[LPL - 1].f[i] += hw.f[i]; Wl[LPL - 1].m[i] += hw.m[i]; }
                    }
                }
            }
            if (K.term_cf >= 0)
                finish_term<MODE>(P, A, sinkB, K.term_cf, gsum<LPF>(jcf), ll, active, p, s_counts, real);

            // Kin(q, o, g, p): FK(q) = T(p) T(g); residuals on every lane of the segment
            if (K.term_kp >= 0 || K.term_kr >= 0) {
                M34 Tp, Tg;
                load_m34(Tp, ipose + 16 * K.kin_inst);
                load_m34(Tg, gT + 16 * K.kin_grasp);
                const M34 Ts = compose(Tp, Tg);
                // position error e = ||t_ee - t*||  (L5)
                const float dx = Tee.t[0] - Ts.t[0], dy = Tee.t[1] - Ts.t[1], dz = Tee.t[2] - Ts.t[2];
                const float e2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                const float epos = sqrtf(e2);
                // rotation error: M = R_ee^T R*, theta = atan2(||vee(M - M^T)||/2, (tr M - 1)/2)  (L4)
                float Mm[9];
#pragma unroll
                for (int i = 0; i < 3; ++i)
#pragma unroll
                    for (int j = 0; j < 3; ++j)
                        Mm[3 * i + j] = fmaf(Tee.r[i], Ts.r[j], fmaf(Tee.r[3 + i], Ts.r[3 + j], Tee.r[6 + i] * Ts.r[6 + j]));
                const float wx = Mm[7] - Mm[5], wy = Mm[2] - Mm[6], wz = Mm[3] - Mm[1];
                const float wn2 = fmaf(wx, wx, fmaf(wy, wy, wz * wz));
                const float wn = sqrtf(wn2);
                const float erot = fatan2_pos(0.5f * wn, 0.5f * (Mm[0] + Mm[4] + Mm[8] - 1.f));
                if (K.term_kp >= 0) finish_term<MODE>(P, A, sinkB, K.term_kp, epos, ll, active, p, s_counts, real);
                if (K.term_kr >= 0) finish_term<MODE>(P, A, sinkB, K.term_kr, erot, ll, active, p, s_counts, real);
                if (GRAD) {
                    Wrench tw;   // on the target placement instance
                    tw.zero();
                    if (K.term_kp >= 0 && epos > 0.f) {
                        const float k = P.term_lam[K.term_kp] / epos;
                        const float fx = dx * k, fy = dy * k, fz = dz * k;      // dJ/dt_ee
                        if (ll == LPF - 1) Wl[LPL - 1].add_point(Tee.t[0], Tee.t[1], Tee.t[2], fx, fy, fz);
                        tw.add_point(Ts.t[0], Ts.t[1], Ts.t[2], -fx, -fy, -fz);
                    }
                    if (K.term_kr >= 0 && wn > 0.f) {
                        // u = R_ee w / ||w||: d theta = -u . omega_ee, +u . omega_target  (Appendix A.2)
                        const float k = P.term_lam[K.term_kr] / wn;
                        const float ux = k * fmaf(Tee.r[0], wx, fmaf(Tee.r[1], wy, Tee.r[2] * wz));
                        const float uy = k * fmaf(Tee.r[3], wx, fmaf(Tee.r[4], wy, Tee.r[5] * wz));
                        const float uz = k * fmaf(Tee.r[6], wx, fmaf(Tee.r[7], wy, Tee.r[8] * wz));
                        if (ll == LPF - 1) { Wl[LPL - 1].m[0] -= ux; Wl[LPL - 1].m[1] -= uy; Wl[LPL - 1].m[2] -= uz; }
                        tw.m[0] += ux; tw.m[1] += uy; tw.m[2] += uz;
                    }
                    const bool movable = P.inst[K.kin_inst].xoff >= 0;
#pragma unroll
                    for (int h = 0; h < HP; ++h) {      // halves add one after the other (deterministic)
                        if (half == h && ll == 0 && real && movable) add_wrench(iwr + 8 * K.kin_inst, tw);
                        if (HP > 1) __syncwarp();
                    }
                }
            }

            // joint limits: dist_from_bounds(q, lo, hi)  (Listing 2; Motion P:1025)
            float ejl[LPL], jl = 0.f;
#pragma unroll
            for (int u = 0; u < LPL; ++u) ejl[u] = 0.f;
            if (K.term_jl >= 0) {
                float e2 = 0.f;
#pragma unroll
                for (int u = 0; u < LPL; ++u) {
                    ejl[u] = ll * LPL + u < TAMP_NJ ? fmaxf(fmaxf(jlo[u] - q[u], q[u] - jhi[u]), 0.f) : 0.f;
                    e2 = fmaf(ejl[u], ejl[u], e2);
                }
                jl = sqrtf(gsum<LPF>(e2));
                finish_term<MODE>(P, A, sinkB, K.term_jl, jl, ll, active, p, s_counts, real);
            }
            if (GRAD) {
                // suffix sums of link wrenches over the links after each joint: dJ/dq_j = z_j . (M - o_j x F)
                Wrench sfx;                               // sum over my links and all later lanes' links
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    sfx.f[i] = Wl[0].f[i] + (LPL == 2 ? Wl[LPL - 1].f[i] : 0.f);
                    sfx.m[i] = Wl[0].m[i] + (LPL == 2 ? Wl[LPL - 1].m[i] : 0.f);
                }
#pragma unroll
                for (int d = 1; d < LPF; d <<= 1) {
                    float v[6];
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        v[i] = __shfl_down_sync(FULL, sfx.f[i], d, LPF);
                        v[3 + i] = __shfl_down_sync(FULL, sfx.m[i], d, LPF);
                    }
                    if (ll + d < LPF) {
#pragma unroll
                        for (int i = 0; i < 3; ++i) { sfx.f[i] += v[i]; sfx.m[i] += v[3 + i]; }
                    }
                }
                Wrench bar[LPL];                          // total wrench on links >= each of my links
                if (LPL == 1) {
                    bar[0] = sfx;
                } else {
                    Wrench nxt;                           // later lanes only
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        nxt.f[i] = __shfl_down_sync(FULL, sfx.f[i], 1, LPF);
                        nxt.m[i] = __shfl_down_sync(FULL, sfx.m[i], 1, LPF);
                        if (ll == LPF - 1) nxt.f[i] = nxt.m[i] = 0.f;
                        bar[LPL - 1].f[i] = Wl[LPL - 1].f[i] + nxt.f[i];
                        bar[LPL - 1].m[i] = Wl[LPL - 1].m[i] + nxt.m[i];
                        bar[0].f[i] = Wl[0].f[i] + bar[LPL - 1].f[i];
                        bar[0].m[i] = Wl[0].m[i] + bar[LPL - 1].m[i];
                    }
                }
#pragma unroll
                for (int u = 0; u < LPL; ++u) {
                    const int j = ll * LPL + u;
                    if (j < TAMP_NJ && real) {
                        const float zx = T[u].r[2], zy = T[u].r[5], zz = T[u].r[8];
                        const float ox = T[u].t[0], oy = T[u].t[1], oz = T[u].t[2];
                        const float mx = bar[u].m[0] - (oy * bar[u].f[2] - oz * bar[u].f[1]);
                        const float my = bar[u].m[1] - (oz * bar[u].f[0] - ox * bar[u].f[2]);
                        const float mz = bar[u].m[2] - (ox * bar[u].f[1] - oy * bar[u].f[0]);
                        float dq = fmaf(zx, mx, fmaf(zy, my, zz * mz));
                        if (K.term_jl >= 0 && jl > 0.f && ejl[u] > 0.f)
                            dq += P.term_lam[K.term_jl] * (q[u] > jhi[u] ? ejl[u] : -ejl[u]) / jl;
                        gs[K.xoff + j] += dq;
                    }
                }
            }
            // keep the block's warps in step through the (large) FK loop body (profiles/README.md):
            // every FK instance (2) or every other one (3)
            if (BSYNC == 2 || (BSYNC == 3 && ((f0 / HP) & 1))) __syncthreads();
        }
        if (BSYNC == 1 || BSYNC == 3) phase_sync();   // all warps leave the FK loop before phase C
        // combine the halves' phase-B terms
        if (HP > 1) {
            sinkB.J += __shfl_xor_sync(FULL, sinkB.J, LPF);
            const unsigned bal = __ballot_sync(FULL, sinkB.sat);
            sinkB.sat = ((bal >> (threadIdx.x & 31 & ~(GS - 1))) & ((1u << GS) - 1u)) == ((1u << GS) - 1u);
        }
        sink.J += sinkB.J;
        sink.sat = sink.sat && sinkB.sat;

        // ---- phase C: StablePlace (support, containment) and CFreePlace per Place ----
        for (int pl = 0; pl < P.n_place; ++pl) {
            const KPlace& Q = P.place[pl];
            const int ii = Q.inst;
            const KInst& I = P.inst[ii];
            const KSurface& Sf = P.surf[Q.surface];
            const float pz = xs[I.xoff + 2];
            Wrench own;
            own.zero();
            // support: |z_bottom - z_top|  (L6; object frame origin at its bottom, L15)
            {
                const float e = fabsf(pz - Sf.frame[2]);
                finish_term<MODE>(P, A, sink, Q.term_ss, e, gl, active, p, s_counts);
                if (GRAD && gl == 0 && e > 0.f) {
                    const float g = P.term_lam[Q.term_ss] * (pz > Sf.frame[2] ? 1.f : -1.f);
                    own.add_point(xs[I.xoff], xs[I.xoff + 1], pz, 0.f, 0.f, g);
                }
            }
            const int no = P.osph_n[I.obj];
            float wq[NSO][3], rq[NSO], gq[NSO][3];
#pragma unroll
            for (int u = 0; u < NSO; ++u) {
                const int k = gl + GS * u;
                const float4 c = k < TAMP_MAX_OBJ_SPHERES ? isph[ii * TAMP_MAX_OBJ_SPHERES + k]   // padded slots: far
                                                          : make_float4(kFar, kFar, kFar, 0.f);
                wq[u][0] = c.x; wq[u][1] = c.y; wq[u][2] = c.z;
                rq[u] = c.w;
                gq[u][0] = gq[u][1] = gq[u][2] = 0.f;
            }
            // containment: sum over spheres of dist_from_bounds(xy in surface frame, lo + r, hi - r)
            {
                float sy, cy;
                fsincos(Sf.frame[3], &sy, &cy);
                float e = 0.f;
#pragma unroll
                for (int u = 0; u < NSO; ++u) {
                    if (gl + GS * u >= no) continue;
                    const float rx = wq[u][0] - Sf.frame[0], ry = wq[u][1] - Sf.frame[1];
                    const float lx = fmaf(cy, rx, sy * ry), ly = fmaf(-sy, rx, cy * ry);
                    const float lox = Sf.lo[0] + rq[u], hix = Sf.hi[0] - rq[u];
                    const float loy = Sf.lo[1] + rq[u], hiy = Sf.hi[1] - rq[u];
                    const float ex = fmaxf(fmaxf(lox - lx, lx - hix), 0.f);
                    const float ey = fmaxf(fmaxf(loy - ly, ly - hiy), 0.f);
                    const float eu = sqrtf(fmaf(ex, ex, ey * ey));
                    e += eu;
                    if (GRAD && eu > 0.f) {
                        const float k = P.term_lam[Q.term_sc] / eu;
                        const float glx = (lx > hix ? ex : (lx < lox ? -ex : 0.f)) * k;
                        const float gly = (ly > hiy ? ey : (ly < loy ? -ey : 0.f)) * k;
                        gq[u][0] += fmaf(cy, glx, -sy * gly);
                        gq[u][1] += fmaf(sy, glx, cy * gly);
                    }
                }
                finish_term<MODE>(P, A, sink, Q.term_sc, gsum<GS>(e), gl, active, p, s_counts);
            }
            // CFreePlace: placed-object spheres vs OBBs (support excluded) and other objects
            {
                const float lam_cp = P.term_lam[Q.term_cp];
                float rqe[NSO];
#pragma unroll
                for (int u = 0; u < NSO; ++u) rqe[u] = rq[u] + P.eta;
                float jcp = 0.f;
                for (int b = 0; b < P.n_obb; ++b)
                    if ((Q.obb_mask >> b) & 1) jcp += spheres_vs_obb<GRAD, NSO>(wq, rqe, P.obb[b], lam_cp, gq);
                for (int pi = 0; pi < Q.part_count; ++pi) {
                    const int jj = P.partners[Q.part_begin + pi];
                    jcp += pairs_vs_instance<GRAD, NSO>(wq, rqe, isph + jj * TAMP_MAX_OBJ_SPHERES, ibound(jj), lam_cp, gq,
                        [&](Wrench& pw) { flush_partner<GRAD, GS>(pw, P.inst[jj].xoff >= 0, iwr + 8 * jj, gl); });
                }
                finish_term<MODE>(P, A, sink, Q.term_cp, gsum<GS>(jcp), gl, active, p, s_counts);
            }
            if (GRAD) {
#pragma unroll
                for (int u = 0; u < NSO; ++u)
                    if (gl + GS * u < no) own.add_point(wq[u][0], wq[u][1], wq[u][2], gq[u][0], gq[u][1], gq[u][2]);
                own.template group_sum<GS>();
                if (gl == 0) add_wrench(iwr + 8 * ii, own);
            }
        }

        // ---- phase D: soft costs (Eq. 2 second sum) ----
        if (P.n_goal > 1) {   // MinimizeObjDist: sum_{i<j} ||P_i - P_j||  (Listing 2 obj_dist)
            for (int a = 0; a < P.n_goal; ++a) {
                for (int b = a + 1; b < P.n_goal; ++b) {
                    const float* pa = ipose + 16 * P.goal_inst[a];
                    const float* pb = ipose + 16 * P.goal_inst[b];
                    const float dx = pa[3] - pb[3], dy = pa[7] - pb[7], dz = pa[11] - pb[11];
                    const float d = sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
                    soft = fmaf(P.lam_goal, d, soft);
                    if (GRAD && gl == 0 && d > 0.f) {
                        const float k = P.lam_goal / d;
                        const int ia = P.goal_inst[a], ib = P.goal_inst[b];
                        if (P.inst[ia].xoff >= 0) {
                            float* t = iwr + 8 * ia;
                            t[0] += dx * k; t[1] += dy * k; t[2] += dz * k;
                            t[3] += pa[7] * dz * k - pa[11] * dy * k;
                            t[4] += pa[11] * dx * k - pa[3] * dz * k;
                            t[5] += pa[3] * dy * k - pa[7] * dx * k;
                        }
                        if (P.inst[ib].xoff >= 0) {
                            float* t = iwr + 8 * ib;
                            t[0] -= dx * k; t[1] -= dy * k; t[2] -= dz * k;
                            t[3] -= pb[7] * dz * k - pb[11] * dy * k;
                            t[4] -= pb[11] * dx * k - pb[3] * dz * k;
                            t[5] -= pb[3] * dy * k - pb[7] * dx * k;
                        }
                    }
                }
            }
        }
        for (int tr = 0; tr < P.n_traj; ++tr) {   // TrajLength(tau) = sum_j ||k_{j+1} - k_j||  (Listing 1 cost)
            const KTraj& Tj = P.traj[tr];
            const int nseg = Tj.n_knots + 1;
            auto val = [&](int j, int jt) -> float {   // j = 0: q1, 1..K: knots, K+1: q2; jt = joint
                if (jt >= TAMP_NJ) return 0.f;
                if (j == 0) return Tj.q1_xoff >= 0 ? xs[Tj.q1_xoff + jt] : P.const_conf[Tj.q1_const][jt];
                if (j == nseg) return Tj.q2_xoff >= 0 ? xs[Tj.q2_xoff + jt] : P.const_conf[Tj.q2_const][jt];
                return xs[Tj.knot_xoff + 7 * (j - 1) + jt];
            };
            auto xoff_of = [&](int j) -> int {
                if (j == 0) return Tj.q1_xoff;
                if (j == nseg) return Tj.q2_xoff;
                return Tj.knot_xoff + 7 * (j - 1);
            };
            for (int j = 0; j < nseg; ++j) {
                float dlt[NJL], s2 = 0.f;
#pragma unroll
                for (int u = 0; u < NJL; ++u) {
                    const int jt = gl + GS * u;
                    dlt[u] = val(j + 1, jt) - val(j, jt);
                    s2 = fmaf(dlt[u], dlt[u], s2);
                }
                const float len = sqrtf(gsum<GS>(s2));
                soft = fmaf(P.lam_traj, len, soft);
                if (GRAD && len > 0.f) {
                    const int o1 = xoff_of(j + 1), o0 = xoff_of(j);
#pragma unroll
                    for (int u = 0; u < NJL; ++u) {
                        const int jt = gl + GS * u;
                        if (jt >= TAMP_NJ) continue;
                        const float g = P.lam_traj * dlt[u] / len;
                        if (o1 >= 0) gs[o1 + jt] += g;
                        if (o0 >= 0) gs[o0 + jt] -= g;
                    }
                }
            }
        }
        const float Jtot = sink.J + soft;

        // ---- phase E: instance wrenches -> placement gradients ----
        if (GRAD) {
            phase_sync();
            for (int i = 0; i < P.n_inst; ++i) {
                const KInst& I = P.inst[i];
                if (I.xoff < 0) continue;
                const float* wr = iwr + 8 * i;
                if (gl < 3) {
                    gs[I.xoff + gl] += wr[gl];
                } else if (gl == 3) {   // d/dyaw = z . (M - t x F)
                    const float tx = xs[I.xoff], ty = xs[I.xoff + 1];
                    gs[I.xoff + 3] += wr[5] - (tx * wr[1] - ty * wr[0]);
                }
            }
            phase_sync();
        }

        if (MODE == MODE_EVAL) {
            if (active) {
                if (gl == 0 && A.out_J) A.out_J[p] = Jtot;
                if (gl == 0 && A.out_soft) A.out_soft[p] = soft;
                if (A.out_grad) for (int d = gl; d < D; d += GS) A.out_grad[p * D + d] = gs[d];
            }
        } else if (MODE == MODE_CHECK) {
            const bool inv = invalid || !isfinite(Jtot);
            const int cls = inv ? 2 : (sink.sat ? 0 : 1);
            if (gl == 0 && active) {
                A.out_cls[p] = (uint8_t)cls;
                A.out_cost[p] = cls == 0 ? soft : (cls == 1 ? Jtot : 0.f);
                if (cls == 0) atomicAdd(&s_counts[P.n_terms], 1);
                if (cls == 2) atomicAdd(&s_counts[P.n_terms + 1], 1);
            }
        } else {
            // ---- phase F: Adam (Kingma & Ba) with grad scale 1/N (Eq. 4) + projection (L11) ----
            bool bad = !isfinite(Jtot);
            for (int d = gl; d < D; d += GS) bad |= !isfinite(gs[d]);
            bad = ((__ballot_sync(FULL, bad) >> (threadIdx.x & 31 & ~(GS - 1))) & ((1u << GS) - 1u)) != 0u;   // my group
            invalid = invalid || bad;
            const float bc1 = A.bc1[it];
            const float bc2 = A.bc2[it];
            if (!invalid) {
                for (int d = gl; d < D; d += GS) {
                    const float g = gs[d] * P.grad_scale;
                    const float mm = fmaf(P.beta1, A.m[p * D + d], (1.f - P.beta1) * g);
                    const float vv = fmaf(P.beta2, A.v[p * D + d], (1.f - P.beta2) * g * g);
                    if (active) { A.m[p * D + d] = mm; A.v[p * D + d] = vv; }
                    const float mh = mm / bc1;
                    const float vh = vv / bc2;
                    const float xn = xs[d] - A.lr[d] * mh / (sqrtf(vh) + P.adam_eps);
                    xs[d] = fminf(fmaxf(xn, A.lo[d]), A.hi[d]);
                }
            }
            phase_sync();
        }
    }

    if (MODE == MODE_OPT && active) {
        for (int d = gl; d < D; d += GS) A.x[p * D + d] = xs[d];
        if (gl == 0) A.invalid[p] = invalid ? 1 : 0;
    }
    if (MODE == MODE_CHECK) {
        __syncthreads();
        for (int i = threadIdx.x; i < P.n_terms + 2; i += blockDim.x)
            if (s_counts[i]) atomicAdd(&A.out_counts[i], s_counts[i]);
    }
}

// ------------------------------------------------------------------------------------------------
// K1: particle initialisation (Philox4x32-10, Salmon et al. SC'11)
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k.x += 0x9E3779B9u; k.y += 0xBB67AE85u; }
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    }
    return c;
}

__device__ __forceinline__ void uniform4(uint64_t seed, uint64_t gidx, int var, int block, float u[4]) {
    const uint4 w = philox4x32_10(make_uint4((uint32_t)gidx, (uint32_t)(gidx >> 32), (uint32_t)var, (uint32_t)block),
                                  make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
    const float s = 1.0f / 16777216.0f;
    u[0] = (float)(w.x >> 8) * s; u[1] = (float)(w.y >> 8) * s;
    u[2] = (float)(w.z >> 8) * s; u[3] = (float)(w.w >> 8) * s;
}

__global__ void __launch_bounds__(128) k_sample(const __grid_constant__ KSampleProgram SP, float* __restrict__ x,
                                                float* __restrict__ grasp, int64_t n, int64_t gofs, uint64_t seed) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t gidx = (uint64_t)(gofs + i);
    float* xi = x + i * SP.D;
    for (int vi = 0; vi < SP.n_vars; ++vi) {
        const KSVar& V = SP.v[vi];
        float u[8];
        if (V.kind == KS_GRASP) {       // top-down grasp: Trans(gx, gy, gz) Rz(gamma) Rx(pi)
            uniform4(seed, gidx, V.var_id, 0, u);
            const float gxy = V.a[0];
            const float gx = -gxy + 2.f * gxy * u[0];
            const float gy = -gxy + 2.f * gxy * u[1];
            const float gamma = -kPi + 2.f * kPi * u[2];
            float s, c;
            sincosf(gamma, &s, &c);
            float* g = grasp + (i * SP.n_grasp + V.slot) * 12;
            g[0] = c;   g[1] = s;   g[2] = 0.f;  g[3] = gx;
            g[4] = s;   g[5] = -c;  g[6] = 0.f;  g[7] = gy;
            g[8] = 0.f; g[9] = 0.f; g[10] = -1.f; g[11] = V.a[1];
        } else if (V.kind == KS_PLACEMENT) {   // uniform on the surface region shrunk by the footprint
            uniform4(seed, gidx, V.var_id, 0, u);
            // a = [region lo x, lo y, hi x, hi y, footprint, frame x, frame y, frame z_top, frame yaw]
            const float wx = fmaxf(V.a[2] - V.a[0] - 2.f * V.a[4], 0.f);
            const float wy = fmaxf(V.a[3] - V.a[1] - 2.f * V.a[4], 0.f);
            const float lx = (V.a[0] + V.a[2]) / 2.f - wx / 2.f + u[0] * wx;
            const float ly = (V.a[1] + V.a[3]) / 2.f - wy / 2.f + u[1] * wy;
            const float lyaw = -kPi + 2.f * kPi * u[2];
            const float fyaw = V.a[8];
            float s, c;
            sincosf(fyaw, &s, &c);
            xi[V.xoff + 0] = V.a[5] + c * lx - s * ly;
            xi[V.xoff + 1] = V.a[6] + s * lx + c * ly;
            xi[V.xoff + 2] = V.a[7];
            xi[V.xoff + 3] = fyaw + lyaw;
        } else if (V.kind == KS_CONF) {        // uniform within joint limits
            uniform4(seed, gidx, V.var_id, 0, u);
            uniform4(seed, gidx, V.var_id, 1, u + 4);
#pragma unroll
            for (int j = 0; j < TAMP_NJ; ++j) xi[V.xoff + j] = SP.jlo[j] + u[j] * (SP.jhi[j] - SP.jlo[j]);
        }
    }
    // knots: linear interpolation between the motion's endpoint confs
    for (int vi = 0; vi < SP.n_vars; ++vi) {
        const KSVar& V = SP.v[vi];
        if (V.kind != KS_TRAJ) continue;
        for (int j = 0; j < V.n_knots; ++j) {
            const float a = (float)(j + 1) / (float)(V.n_knots + 1);
            for (int d = 0; d < TAMP_NJ; ++d) {
                const float qa = V.q1_xoff >= 0 ? xi[V.q1_xoff + d] : SP.const_conf[V.q1_const][d];
                const float qb = V.q2_xoff >= 0 ? xi[V.q2_xoff + d] : SP.const_conf[V.q2_const][d];
                xi[V.xoff + 7 * j + d] = qa + a * (qb - qa);
            }
        }
    }
}

// ------------------------------------------------------------------------------------------------
// K1b: conditional IK sampler -- damped least squares toward each Pick/Place conf's Kin target
// T(p) T(g), one particle per 8-lane group (lane j = joint j+1, the same FK product scan as K2), then the
// knots are re-interpolated from the refined endpoint confs.
//   e = [t* - t_ee ; rotvec(R* R_ee^T)],  J = [z_j x (t_ee - o_j) ; z_j],  dq = J^T (J J^T + mu^2 I)^-1 e
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ void chol6_solve(float A[21], const float b[6], float y[6]) {
    // A: packed lower triangle, row-major (i, j <= i) -> index i*(i+1)/2 + j.  In-place Cholesky.
#pragma unroll
    for (int j = 0; j < 6; ++j) {
        float d = A[j * (j + 1) / 2 + j];
#pragma unroll
        for (int k = 0; k < j; ++k) d = fmaf(-A[j * (j + 1) / 2 + k], A[j * (j + 1) / 2 + k], d);
        const float ljj = sqrtf(fmaxf(d, 1e-30f));
        const float inv = 1.f / ljj;
        A[j * (j + 1) / 2 + j] = ljj;
#pragma unroll
        for (int i = j + 1; i < 6; ++i) {
            float v = A[i * (i + 1) / 2 + j];
#pragma unroll
            for (int k = 0; k < j; ++k) v = fmaf(-A[i * (i + 1) / 2 + k], A[j * (j + 1) / 2 + k], v);
            A[i * (i + 1) / 2 + j] = v * inv;
        }
    }
    float z[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) {     // L z = b
        float v = b[i];
#pragma unroll
        for (int k = 0; k < i; ++k) v = fmaf(-A[i * (i + 1) / 2 + k], z[k], v);
        z[i] = v / A[i * (i + 1) / 2 + i];
    }
#pragma unroll
    for (int i = 5; i >= 0; --i) {    // L^T y = z
        float v = z[i];
#pragma unroll
        for (int k = i + 1; k < 6; ++k) v = fmaf(-A[k * (k + 1) / 2 + i], y[k], v);
        y[i] = v / A[i * (i + 1) / 2 + i];
    }
}

__global__ void __launch_bounds__(128) k_ik(const __grid_constant__ KProgram P, float* __restrict__ x,
                                            const float* __restrict__ grasp, int64_t n, int iters, float damp2) {
    const int gl = threadIdx.x & (kGroup - 1);
    const int64_t pid = (int64_t)blockIdx.x * (blockDim.x / kGroup) + threadIdx.x / kGroup;
    const bool active = pid < n;
    const int64_t p = active ? pid : (n - 1);
    const int D = P.D;
    float* xp = x + p * D;
    M34 F;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        F.r[3 * i] = P.F[gl][4 * i]; F.r[3 * i + 1] = P.F[gl][4 * i + 1];
        F.r[3 * i + 2] = P.F[gl][4 * i + 2]; F.t[i] = P.F[gl][4 * i + 3];
    }
    const float jlo = gl < TAMP_NJ ? P.jlo[gl] : 0.f;
    const float jhi = gl < TAMP_NJ ? P.jhi[gl] : 0.f;
    for (int f = 0; f < P.n_fk; ++f) {
        const KFk K = P.fk[f];
        if ((K.term_kp < 0 && K.term_kr < 0) || K.ghost) continue;
        // Kin target T* = T(p) T(g)
        const KInst& I = P.inst[K.kin_inst];
        float pp[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) pp[k] = I.xoff >= 0 ? xp[I.xoff + k] : I.pose[k];
        float sy, cy;
        fsincos(pp[3], &sy, &cy);
        M34 Tp, Tg;
        Tp.r[0] = cy; Tp.r[1] = -sy; Tp.r[2] = 0.f; Tp.r[3] = sy; Tp.r[4] = cy; Tp.r[5] = 0.f;
        Tp.r[6] = 0.f; Tp.r[7] = 0.f; Tp.r[8] = 1.f; Tp.t[0] = pp[0]; Tp.t[1] = pp[1]; Tp.t[2] = pp[2];
        load_m34(Tg, grasp + (p * P.n_grasp + K.kin_grasp) * 12);
        const M34 Ts = compose(Tp, Tg);
        float q = gl < TAMP_NJ ? xp[K.xoff + gl] : 0.f;
        for (int it = 0; it < iters; ++it) {
            M34 T;
            {
                float s, c;
                fsincos(q, &s, &c);
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    T.r[3 * i] = fmaf(F.r[3 * i], c, F.r[3 * i + 1] * s);
                    T.r[3 * i + 1] = fmaf(F.r[3 * i + 1], c, -F.r[3 * i] * s);
                    T.r[3 * i + 2] = F.r[3 * i + 2];
                    T.t[i] = F.t[i];
                }
            }
#pragma unroll
            for (int d = 1; d < kGroup; d <<= 1) {
                const M34 U = shfl_up_m34(T, d);
                if (gl >= d) T = compose(U, T);
            }
            const M34 Tee = shfl_m34(T, kGroup - 1);
            float e[6];
            e[0] = Ts.t[0] - Tee.t[0]; e[1] = Ts.t[1] - Tee.t[1]; e[2] = Ts.t[2] - Tee.t[2];
            float E[9];   // R* R_ee^T
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int j = 0; j < 3; ++j)
                    E[3 * i + j] = fmaf(Ts.r[3 * i], Tee.r[3 * j], fmaf(Ts.r[3 * i + 1], Tee.r[3 * j + 1], Ts.r[3 * i + 2] * Tee.r[3 * j + 2]));
            const float wx = E[7] - E[5], wy = E[2] - E[6], wz = E[3] - E[1];
            const float wn = sqrtf(fmaf(wx, wx, fmaf(wy, wy, wz * wz)));
            const float th = atan2f(0.5f * wn, 0.5f * (E[0] + E[4] + E[8] - 1.f));
            const float k = wn > 0.f ? th / wn : 0.f;
            e[3] = wx * k; e[4] = wy * k; e[5] = wz * k;
            // Jacobian column of my joint
            float c[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            if (gl < TAMP_NJ) {
                const float zx = T.r[2], zy = T.r[5], zz = T.r[8];
                const float rx = Tee.t[0] - T.t[0], ry = Tee.t[1] - T.t[1], rz = Tee.t[2] - T.t[2];
                c[0] = zy * rz - zz * ry; c[1] = zz * rx - zx * rz; c[2] = zx * ry - zy * rx;
                c[3] = zx; c[4] = zy; c[5] = zz;
            }
            float A[21];
#pragma unroll
            for (int i = 0; i < 6; ++i)
#pragma unroll
                for (int j = 0; j <= i; ++j) A[i * (i + 1) / 2 + j] = gsum<kGroup>(c[i] * c[j]) + (i == j ? damp2 : 0.f);
            float y[6];
            chol6_solve(A, e, y);
            const float dq = fmaf(c[0], y[0], fmaf(c[1], y[1], fmaf(c[2], y[2], fmaf(c[3], y[3], fmaf(c[4], y[4], c[5] * y[5])))));
            if (gl < TAMP_NJ) q = fminf(fmaxf(q + dq, jlo), jhi);
        }
        if (gl < TAMP_NJ && active) xp[K.xoff + gl] = q;
        __syncwarp();
    }
    // knots: linear interpolation between the (refined) endpoint confs
    for (int tr = 0; tr < P.n_traj; ++tr) {
        const KTraj& Tj = P.traj[tr];
        if (gl >= TAMP_NJ || !active) continue;
        const float qa = Tj.q1_xoff >= 0 ? xp[Tj.q1_xoff + gl] : P.const_conf[Tj.q1_const][gl];
        const float qb = Tj.q2_xoff >= 0 ? xp[Tj.q2_xoff + gl] : P.const_conf[Tj.q2_const][gl];
        for (int j = 0; j < Tj.n_knots; ++j) {
            const float a = (float)(j + 1) / (float)(Tj.n_knots + 1);
            xp[Tj.knot_xoff + 7 * j + gl] = qa + a * (qb - qa);
        }
    }
}

// ------------------------------------------------------------------------------------------------
// K4 / K5: best-k (key = class | ordered cost | global index)
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t ordered_bits(float f) {
    const uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ unsigned long long make_key(int cls, float cost, int64_t gidx) {
    return ((unsigned long long)(cls & 3) << 62) | ((unsigned long long)ordered_bits(cost) << 30) |
           ((unsigned long long)gidx & ((1ull << 30) - 1));
}

constexpr int kSortChunk = 2048;

// keys from the check pass (payload = local particle index)
__global__ void k_make_keys(const uint8_t* __restrict__ cls, const float* __restrict__ cost, int64_t n, int64_t gofs,
                            unsigned long long* __restrict__ keys, int32_t* __restrict__ pay) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    keys[i] = make_key(cls[i], cost[i], gofs + i);
    pay[i] = (int32_t)i;
}

// keys from gathered records [class, cost, gidx_lo, gidx_hi, x...] (payload = record row)
__global__ void k_record_keys(const float* __restrict__ rec, int32_t n, int32_t width,
                              unsigned long long* __restrict__ keys, int32_t* __restrict__ pay) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float* r = rec + (int64_t)i * width;
    const int64_t gidx = (int64_t)(uint32_t)__float_as_int(r[2]) | ((int64_t)__float_as_int(r[3]) << 32);
    keys[i] = make_key((int)r[0], r[1], gidx);
    pay[i] = i;
}

// Sort each chunk of kSortChunk (key, payload) pairs ascending and keep its first k.
__global__ void __launch_bounds__(1024) k_sort_chunk(const unsigned long long* __restrict__ kin, const int32_t* __restrict__ pin,
                                                     int64_t n, int k, unsigned long long* __restrict__ kout,
                                                     int32_t* __restrict__ pout) {
    __shared__ unsigned long long sk[kSortChunk];
    __shared__ int32_t sp[kSortChunk];
    const int64_t base = (int64_t)blockIdx.x * kSortChunk;
    for (int i = threadIdx.x; i < kSortChunk; i += blockDim.x) {
        const int64_t g = base + i;
        sk[i] = g < n ? kin[g] : ~0ull;
        sp[i] = g < n ? pin[g] : -1;
    }
    __syncthreads();
    for (int size = 2; size <= kSortChunk; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < kSortChunk / 2; i += blockDim.x) {
                const int lo = 2 * i - (i & (stride - 1));
                const int hi = lo + stride;
                const bool up = ((lo & size) == 0);
                const unsigned long long a = sk[lo], b = sk[hi];
                if ((a > b) == up) {
                    sk[lo] = b; sk[hi] = a;
                    const int32_t t = sp[lo]; sp[lo] = sp[hi]; sp[hi] = t;
                }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
        kout[(int64_t)blockIdx.x * k + i] = sk[i];
        pout[(int64_t)blockIdx.x * k + i] = sp[i];
    }
}

__global__ void k_gather_particles(const int32_t* __restrict__ pay, const unsigned long long* __restrict__ keys, int k,
                                   const float* __restrict__ x, const float* __restrict__ cost, int D, int64_t gofs,
                                   float* __restrict__ rec) {
    const int r = blockIdx.x;
    if (r >= k) return;
    const int32_t i = pay[r];
    float* o = rec + (int64_t)r * (D + 4);
    if (threadIdx.x == 0) {
        const int64_t gidx = gofs + i;
        o[0] = (float)(int)(keys[r] >> 62);
        o[1] = cost[i];
        o[2] = __int_as_float((int32_t)(uint32_t)(gidx & 0xffffffffll));
        o[3] = __int_as_float((int32_t)(gidx >> 32));
    }
    for (int d = threadIdx.x; d < D; d += blockDim.x) o[4 + d] = x[(int64_t)i * D + d];
}

__global__ void k_gather_records(const int32_t* __restrict__ pay, int k, const float* __restrict__ rin, int width,
                                 float* __restrict__ rout) {
    const int r = blockIdx.x;
    if (r >= k) return;
    const float* s = rin + (int64_t)pay[r] * width;
    for (int d = threadIdx.x; d < width; d += blockDim.x) rout[(int64_t)r * width + d] = s[d];
}

// ------------------------------------------------------------------------------------------------
// launchers (called from tamp_api.cu)
// ------------------------------------------------------------------------------------------------
static std::atomic<uint64_t> g_launches{0};
uint64_t launch_count() { return g_launches.load(); }
static inline void counted() { g_launches.fetch_add(1, std::memory_order_relaxed); }

template <int MODE, int LPF, int HP, int BSYNC>
static cudaError_t launch_particle_t(const KProgram& P, const KArgs& A, int threads, size_t smem, cudaStream_t st) {
    auto fn = k_particle<MODE, LPF, HP, BSYNC>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int per_block = threads / (LPF * HP);
    const int64_t blocks = (A.n + per_block - 1) / per_block;
    fn<<<(unsigned)blocks, threads, smem, st>>>(P, A);
    counted();
    return cudaGetLastError();
}

template <int LPF, int HP>
static cudaError_t launch_particle_map(int mode, int bsync, const KProgram& P, const KArgs& A, int threads, size_t smem,
                                       cudaStream_t st) {
    if (mode == MODE_EVAL) return launch_particle_t<MODE_EVAL, LPF, HP, 2>(P, A, threads, smem, st);
    if (mode == MODE_CHECK) {
        if (bsync == 0) return launch_particle_t<MODE_CHECK, LPF, HP, 0>(P, A, threads, smem, st);
        if (bsync == 1) return launch_particle_t<MODE_CHECK, LPF, HP, 1>(P, A, threads, smem, st);
        return launch_particle_t<MODE_CHECK, LPF, HP, 2>(P, A, threads, smem, st);
    }
    switch (bsync) {
        case 0: return launch_particle_t<MODE_OPT, LPF, HP, 0>(P, A, threads, smem, st);
        case 1: return launch_particle_t<MODE_OPT, LPF, HP, 1>(P, A, threads, smem, st);
        case 3: return launch_particle_t<MODE_OPT, LPF, HP, 3>(P, A, threads, smem, st);
        default: return launch_particle_t<MODE_OPT, LPF, HP, 2>(P, A, threads, smem, st);
    }
}

// registers per thread of the hot kernel (for the launch-configuration policy)
int particle_kernel_regs(int gs) {
    cudaFuncAttributes a;
    cudaError_t e = gs == 16 ? cudaFuncGetAttributes(&a, k_particle<MODE_OPT, 8, 2, 1>)
                  : gs == 4  ? cudaFuncGetAttributes(&a, k_particle<MODE_OPT, 4, 1, 1>)
                             : cudaFuncGetAttributes(&a, k_particle<MODE_OPT, 8, 1, 1>);
    if (e != cudaSuccess) { cudaGetLastError(); return 80; }
    return a.numRegs;
}

// gs = lanes per particle: 4 (two link frames per lane), 8 (one), 16 (two FK instances at a time);
// threads = block size (multiple of 32, <= 768); smem sized for threads / gs particles;
// bsync = block-synchronisation level (see k_particle).
cudaError_t launch_particle(int mode, int gs, int bsync, int threads, const KProgram& P, const KArgs& A, size_t smem,
                            cudaStream_t st) {
    if (A.n <= 0) return cudaSuccess;
    if (gs == 16) return launch_particle_map<8, 2>(mode, bsync, P, A, threads, smem, st);
    if (gs == 4) return launch_particle_map<4, 1>(mode, bsync, P, A, threads, smem, st);
    return launch_particle_map<8, 1>(mode, bsync, P, A, threads, smem, st);
}

cudaError_t launch_ik(const KProgram& P, float* x, const float* grasp, int64_t n, int iters, float damping,
                      cudaStream_t st) {
    if (n <= 0 || iters <= 0) return cudaSuccess;
    const int per_block = 128 / kGroup;
    k_ik<<<(unsigned)((n + per_block - 1) / per_block), 128, 0, st>>>(P, x, grasp, n, iters, damping * damping);
    counted();
    return cudaGetLastError();
}

cudaError_t launch_sample(const KSampleProgram& SP, float* x, float* grasp, int64_t n, int64_t gofs, uint64_t seed,
                          cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    k_sample<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(SP, x, grasp, n, gofs, seed);
    counted();
    return cudaGetLastError();
}

// top-k of n (key, payload) pairs in ka/pa (ping-pong with kb/pb).  Returns pointers to the result.
cudaError_t launch_topk(unsigned long long* ka, int32_t* pa, unsigned long long* kb, int32_t* pb, int64_t n, int k,
                        cudaStream_t st, unsigned long long** kres, int32_t** pres) {
    unsigned long long *ki = ka, *ko = kb;
    int32_t *pi = pa, *po = pb;
    int64_t cnt = n;
    do {
        const int64_t chunks = (cnt + kSortChunk - 1) / kSortChunk;
        const int keep = (int)(cnt < k ? cnt : k);
        k_sort_chunk<<<(unsigned)chunks, 1024, 0, st>>>(ki, pi, cnt, keep, ko, po);
    counted();
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        cnt = chunks * keep;
        unsigned long long* t = ki; ki = ko; ko = t;
        int32_t* u = pi; pi = po; po = u;
        if (chunks == 1) break;
    } while (true);
    *kres = ki;
    *pres = pi;
    return cudaSuccess;
}

cudaError_t launch_make_keys(const uint8_t* cls, const float* cost, int64_t n, int64_t gofs, unsigned long long* keys,
                             int32_t* pay, cudaStream_t st) {
    k_make_keys<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(cls, cost, n, gofs, keys, pay);
    counted();
    return cudaGetLastError();
}

cudaError_t launch_record_keys(const float* rec, int32_t n, int32_t width, unsigned long long* keys, int32_t* pay,
                               cudaStream_t st) {
    k_record_keys<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(rec, n, width, keys, pay);
    counted();
    return cudaGetLastError();
}

cudaError_t launch_gather_particles(const int32_t* pay, const unsigned long long* keys, int k, const float* x,
                                    const float* cost, int D, int64_t gofs, float* rec, cudaStream_t st) {
    k_gather_particles<<<k, 128, 0, st>>>(pay, keys, k, x, cost, D, gofs, rec);
    counted();
    return cudaGetLastError();
}

cudaError_t launch_gather_records(const int32_t* pay, int k, const float* rin, int width, float* rout, cudaStream_t st) {
    k_gather_records<<<k, 128, 0, st>>>(pay, k, rin, width, rout);
    counted();
    return cudaGetLastError();
}

}  // namespace tamp
