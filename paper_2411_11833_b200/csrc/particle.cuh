// particle.cuh -- device helpers and the fused per-particle kernel template k_particle (K2 / K3 / eval).
// Included by tamp_kernels.cu (helpers for K1b) and by the two instantiation units
// tamp_particle_hinge.cu / tamp_particle_smooth.cu (compiled in parallel).
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <type_traits>

#include "tamp_program.h"

// build-time variants of the sphere tests (A/B experiments, tools/build_variants.py; the defaults are the product):
//   TAMP_PACK_XFORM   1: robot sphere centres transformed in packed pairs (FFMA2), 0: scalar
//   TAMP_PACK_OBB     0: scalar sphere-box reject test (FMNMX), 1: packed pairs with a + |a| on the FMA pipe,
//                     2: packed offsets / rotation, scalar max
//   TAMP_PACK_NARROW  1: sphere-sphere pair tests in packed pairs (one predicate, bit masks only on a hit), 0: scalar
#ifndef TAMP_PACK_XFORM
#define TAMP_PACK_XFORM 1
#endif
#ifndef TAMP_PACK_OBB
#define TAMP_PACK_OBB 1
#endif
#ifndef TAMP_PACK_NARROW
#define TAMP_PACK_NARROW 1
#endif
#ifndef TAMP_PARTNER_TABLE         // lane mappings: partner references as shared-memory offset words in the
#define TAMP_PARTNER_TABLE 1       // register-rich (512-bound) variants: config 2 -2.7 %; the 768 / 896-bound ones
#endif                             // were slower with it (config 4 +1.5 %, config 3 +0.6 %)
#ifndef TAMP_PLACE_PIN            // lane mappings: the Place descriptor's fields pinned in registers
#define TAMP_PLACE_PIN 1
#endif
#ifndef TAMP_FK_COPY              // with TAMP_FK_SMEM: a register copy of the shared descriptor (else a reference:
#define TAMP_FK_COPY 1            // re-read after every shared-memory store; config 4 7.59 -> 7.18 ms, config 2 -1.2 %)
#endif
#ifndef TAMP_FK_SMEM_MAXT         // variants (launch bound <= this) that read the descriptors from shared memory
#define TAMP_FK_SMEM_MAXT 1024    // (with the register copy also the 896 / 1024-bound ones: config 3 -0.5 %)
#endif
#ifndef TAMP_FK_SMEM              // lane mappings: the configurations' descriptors in the block's shared constant
#define TAMP_FK_SMEM 1            // area (variants with a launch bound <= TAMP_FK_SMEM_MAXT)
#endif
#ifndef TAMP_OBB_SMEM             // lane mappings: boxes' fast-path data staged in shared memory once per block
#define TAMP_OBB_SMEM 1           // (config 3 -0.3 %, config 4 -1.4 % per launch)
#endif
#ifndef TAMP_ROLLED_HITS          // spheres_vs_obb: the exact hinges of the hit spheres as one rolled loop in the
#define TAMP_ROLLED_HITS 1        // 16-lane variants (config 4: 8.13 -> 7.90 ms per launch); the 8-lane 896-thread
#endif                            // variant (72 registers) was slower with it (config 3: 1.81 -> 1.91 ms)
#ifndef TAMP_BOX_CORNER         // aligned boxes: the conservative corner-form reject test (obb_reach_corner_pair)
#define TAMP_BOX_CORNER 1
#endif
#ifndef TAMP_FUNNEL_MASK        // active-pair masks built with one funnel shift per pair (instance_pair_tests)
#define TAMP_FUNNEL_MASK 1
#endif
static_assert(TAMP_MAX_OBJ_SPHERES <= 32, "active-pair masks hold one bit per partner sphere");

// TAMP_DEVICE_CHECKS=1 (tools/device_checks.sh): device-side bounds checks of the shared-memory carve-outs and the
// program's indices, trapping with a message (compute-sanitizer is not available on the GPU pool)
#ifndef TAMP_DEVICE_CHECKS
#define TAMP_DEVICE_CHECKS 0
#endif
#if TAMP_DEVICE_CHECKS
#include <cstdio>
#define TAMP_DCHECK(c)                                                                                    \
    do {                                                                                                  \
        if (!(c)) {                                                                                       \
            printf("TAMP_DCHECK failed: %s (%s:%d) block %d thread %d\n", #c, __FILE__, __LINE__,          \
                   (int)blockIdx.x, (int)threadIdx.x);                                                    \
            __trap();                                                                                     \
        }                                                                                                 \
    } while (0)
#else
#define TAMP_DCHECK(c) do { } while (0)
#endif

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

// T(p) T(g) for a placement T(p) = (Rz(yaw), t) stored as the 3x4 rows of ipose (cos at [0], sin at [4]):
// rows 0 / 1 of the rotation mix, row 2 is T(g)'s
__device__ __forceinline__ M34 compose_rz(const float* ip, const M34& b) {
    const float c = ip[0], s = ip[4];
    M34 o;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        o.r[j] = fmaf(c, b.r[j], -s * b.r[3 + j]);
        o.r[3 + j] = fmaf(s, b.r[j], c * b.r[3 + j]);
        o.r[6 + j] = b.r[6 + j];
    }
    o.t[0] = fmaf(c, b.t[0], fmaf(-s, b.t[1], ip[3]));
    o.t[1] = fmaf(s, b.t[0], fmaf(c, b.t[1], ip[7]));
    o.t[2] = b.t[2] + ip[11];
    return o;
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

// opaque register copies: the compiler cannot re-derive the value (e.g. re-load it from the constant bank)
__device__ __forceinline__ int opaque_int(int v) { asm volatile("" : "+r"(v)); return v; }
__device__ __forceinline__ float opaque_f(float v) { asm volatile("" : "+f"(v)); return v; }

// 4-byte asynchronous copy global -> shared (cp.async.ca; completed by cp_async_wait_all)
__device__ __forceinline__ void cp_async4(float* smem_dst, const float* gsrc) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// MUFU approximations without the denormal rescaling of sqrtf / division under -prec-sqrt=false / -prec-div=false
// (inputs here are >= 0 Adam second moments and sums >= adam_eps > 0)
__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
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
// smoothed collision cost (CHOMP): p -> p - s/2 (p > s), p^2/(2 s) (0 < p <= s); returns the cost and
// sets `gsc` to dcost/dp.  s = 0: plain hinge.
__device__ __forceinline__ float smooth_cost(float p, float s, float& gsc) {
    gsc = 1.f;
    if (s > 0.f) {   // s is the literal 0 in the hinge instantiations: folded away
        gsc = fminf(p / s, 1.f);
        p = p < s ? 0.5f * p * p / s : p - 0.5f * s;
    }
    return p;
}

// ALIGNED: the caller guarantees B.aligned (R = I): the rotations are omitted (the same values)
template <bool GRAD, bool ALIGNED = false>
__device__ __forceinline__ float sphere_obb(float wx, float wy, float wz, float rr, const KObb& B, float lam,
                                            float& gx, float& gy, float& gz, float smooth = 0.f) {
    // oriented box: p = R^T (w - c) with R the box's full rotation (row-major); for a box yawed
    // about z (R[2] = R[5] = R[6] = R[7] = 0, R[8] = 1) the extra terms are exact zeros
    const float dx = wx - B.c[0], dy = wy - B.c[1], dz = wz - B.c[2];
    float px = dx, py = dy, pz = dz;                     // axis-aligned box: R = I (the same values, exactly)
    if (!ALIGNED && !B.aligned) {
        px = fmaf(B.R[0], dx, fmaf(B.R[3], dy, B.R[6] * dz));
        py = fmaf(B.R[1], dx, fmaf(B.R[4], dy, B.R[7] * dz));
        pz = fmaf(B.R[2], dx, fmaf(B.R[5], dy, B.R[8] * dz));
    }
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
    float pen = rr - sd;
    if (!(pen > 0.f)) return 0.f;
    float gsc;
    pen = smooth_cost(pen, smooth, gsc);
    lam *= gsc;
    if (GRAD && ALIGNED) {   // R = I
        gx = fmaf(-lam, gpx, gx);
        gy = fmaf(-lam, gpy, gy);
        gz = fmaf(-lam, gpz, gz);
    } else if (GRAD) {   // dJ/dw = -R grad_p
        gx = fmaf(-lam, fmaf(B.R[0], gpx, fmaf(B.R[1], gpy, B.R[2] * gpz)), gx);
        gy = fmaf(-lam, fmaf(B.R[3], gpx, fmaf(B.R[4], gpy, B.R[5] * gpz)), gy);
        gz = fmaf(-lam, fmaf(B.R[6], gpx, fmaf(B.R[7], gpy, B.R[8] * gpz)), gz);
    }
    return pen;
}

// Can a sphere (centre w, radius r) reach the OBB?  false only if it is outside the box and its centre is at
// least r from it -- the exact test sphere_obb rejects on, so a bounding sphere that fails it bounds only
// spheres whose hinges are all zero.
template <bool ALIGNED = false>
__device__ __forceinline__ bool obb_within(float wx, float wy, float wz, float r, const KObb& B) {
    const float dx = wx - B.c[0], dy = wy - B.c[1], dz = wz - B.c[2];
    float px = dx, py = dy, pz = dz;                     // axis-aligned box: R = I (the same values, exactly)
    if (!ALIGNED && !B.aligned) {
        px = fmaf(B.R[0], dx, fmaf(B.R[3], dy, B.R[6] * dz));
        py = fmaf(B.R[1], dx, fmaf(B.R[4], dy, B.R[7] * dz));
        pz = fmaf(B.R[2], dx, fmaf(B.R[5], dy, B.R[8] * dz));
    }
    const float ax = fabsf(px) - B.h[0], ay = fabsf(py) - B.h[1], az = fabsf(pz) - B.h[2];
    const float qx = fmaxf(ax, 0.f), qy = fmaxf(ay, 0.f), qz = fmaxf(az, 0.f);
    const float s = fmaf(qx, qx, fmaf(qy, qy, qz * qz));
    return !(fmaxf(ax, fmaxf(ay, az)) > 0.f && s >= r * r);
}
// slack added to a link's bounding radius in the link-level broad phase: covers the fp32 difference between
// transforming the link's bounding centre and its sphere centres (~1e-7 m at arm scale)
constexpr float kLinkMargin = 1e-5f;

// Sphere vs sphere.  Returns the hinge; if GRAD: (ux, uy, uz) = lam * (w_a - w_b)/||.|| (0 if inactive).
template <bool GRAD>
__device__ __forceinline__ float sphere_sphere(float ax, float ay, float az, float rr, float4 b,
                                               float lam, float& ux, float& uy, float& uz, float smooth = 0.f) {
    const float dx = ax - b.x, dy = ay - b.y, dz = az - b.z;
    const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    const float R = rr + b.w;
    ux = uy = uz = 0.f;
    if (fmaf(-R, R, d2) >= 0.f) return 0.f;
    float gsc;
    if (d2 > 0.f) {
        const float inv = rsqrtf(d2);
        float pen = R - d2 * inv;
        if (!(pen > 0.f)) return 0.f;
        pen = smooth_cost(pen, smooth, gsc);
        if (GRAD) {
            const float k = lam * gsc * inv;
            ux = dx * k; uy = dy * k; uz = dz * k;
        }
        return pen;
    }
    return smooth_cost(R, smooth, gsc);   // coincident centres: zero gradient (L13)
}

constexpr float kFar = 1e18f;   // position of padded (absent) spheres: never within reach of anything
// OBBs whose bounding sphere is at least this large skip the bounding-sphere broad phase.  0: no box uses it -- with
// the packed exact reject test (about 6 issued instructions per sphere) a thin wall's bounding sphere passed for
// two thirds of the tests and only added work (config 3: 1.89 -> 1.85 ms per launch, profiles/README.md)
#ifndef TAMP_BROAD_MAX_RAD
#define TAMP_BROAD_MAX_RAD 0.0f
#endif
constexpr float kBroadMaxRad = TAMP_BROAD_MAX_RAD;
#ifndef TAMP_NARROW_UNROLL
#define TAMP_NARROW_UNROLL 2
#endif
constexpr int kNarrowUnroll = TAMP_NARROW_UNROLL;     // unrolling of the partner-sphere loop of the pair tests

// ------------------------------------------------------------------------------------------------
// packed fp32x2 arithmetic: FADD2 / FMUL2 / FFMA2 of sm_100a do two IEEE fp32 operations (round to nearest, each
// half exactly the scalar FADD / FMUL / FFMA) in one issued instruction; a scalar operand packed as {a, a} is a
// free broadcast.  The sphere tests below run on pairs of spheres: half the issue slots of the scalar code with
// bit-identical results (measured issue rates on the B200: 3.8 FFMA vs 2.0 FFMA2 warp-instructions per cycle per
// SM, i.e. the same FMA throughput for half the issue slots; tools/micro/pipe_rate.cu)
// ------------------------------------------------------------------------------------------------
struct F2 {
    unsigned long long v;
};
__device__ __forceinline__ F2 pk(float a, float b) {
    F2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ F2 bc(float a) { return pk(a, a); }
__device__ __forceinline__ float lo(F2 x) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(x.v));
    return a;
}
__device__ __forceinline__ float hi(F2 x) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(x.v));
    return b;
}
__device__ __forceinline__ F2 add2(F2 a, F2 b) {
    F2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
    return r;
}
__device__ __forceinline__ F2 sub2(F2 a, F2 b) {
    F2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
    return r;
}
__device__ __forceinline__ F2 mul2(F2 a, F2 b) {
    F2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
    return r;
}
__device__ __forceinline__ F2 fma2(F2 a, F2 b, F2 c) {
    F2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(a.v), "l"(b.v), "l"(c.v));
    return r;
}
// |d|^2 - R^2 with R = ra + rb, as fmaf(-R, R, |d|^2) per half (the scalar code's exact reject quantity);
// -R = (-rb) - ra is exact, and both negations fold into the FADD2's operand modifiers
__device__ __forceinline__ F2 reach2(F2 dx, F2 dy, F2 dz, F2 ra, float rb) {
    return fma2(add2(ra, bc(rb)), sub2(bc(-rb), ra), fma2(dx, dx, fma2(dy, dy, mul2(dz, dz))));
}

// A rigid transform (3x4) with rows 0 and 1 packed: r01[k] = (R[0][k], R[1][k]), t01 = (t0, t1); row 2 scalar.
// compose / xform / the joint-angle rotation run rows 0-1 as FFMA2 with broadcast entries of the right operand, in
// the scalar code's operation order (same values): 24 issued instructions per compose instead of 36.
struct M34P {
    F2 r01[3];
    F2 t01;
    float r2[3];
    float t2;
    __device__ __forceinline__ float r(int i, int k) const {
        return i == 0 ? lo(r01[k]) : (i == 1 ? hi(r01[k]) : r2[k]);
    }
    __device__ __forceinline__ float t(int i) const { return i == 0 ? lo(t01) : (i == 1 ? hi(t01) : t2); }
};
__device__ __forceinline__ M34P pack_m34(const M34& a) {
    M34P o;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        o.r01[k] = pk(a.r[k], a.r[3 + k]);
        o.r2[k] = a.r[6 + k];
    }
    o.t01 = pk(a.t[0], a.t[1]);
    o.t2 = a.t[2];
    return o;
}
__device__ __forceinline__ M34 unpack_m34(const M34P& a) {
    M34 o;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
#pragma unroll
        for (int k = 0; k < 3; ++k) o.r[3 * i + k] = a.r(i, k);
        o.t[i] = a.t(i);
    }
    return o;
}
// a * b (b scalar: its entries are broadcast operands)
__device__ __forceinline__ M34P compose_p(const M34P& a, const M34& b) {
    M34P c;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        c.r01[j] = fma2(a.r01[0], bc(b.r[j]), fma2(a.r01[1], bc(b.r[3 + j]), mul2(a.r01[2], bc(b.r[6 + j]))));
        c.r2[j] = fmaf(a.r2[0], b.r[j], fmaf(a.r2[1], b.r[3 + j], a.r2[2] * b.r[6 + j]));
    }
    c.t01 = fma2(a.r01[0], bc(b.t[0]), fma2(a.r01[1], bc(b.t[1]), fma2(a.r01[2], bc(b.t[2]), a.t01)));
    c.t2 = fmaf(a.r2[0], b.t[0], fmaf(a.r2[1], b.t[1], fmaf(a.r2[2], b.t[2], a.t2)));
    return c;
}
__device__ __forceinline__ M34P shfl_up_m34p(const M34P& a, int d, int width) {
    M34P o;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        o.r01[k] = pk(__shfl_up_sync(FULL, lo(a.r01[k]), d, width), __shfl_up_sync(FULL, hi(a.r01[k]), d, width));
        o.r2[k] = __shfl_up_sync(FULL, a.r2[k], d, width);
    }
    o.t01 = pk(__shfl_up_sync(FULL, lo(a.t01), d, width), __shfl_up_sync(FULL, hi(a.t01), d, width));
    o.t2 = __shfl_up_sync(FULL, a.t2, d, width);
    return o;
}
// Modified-DH link step on the packed frame (columns X = (r01[0], r2[0]), Y, Z, origin o):
// T_j = T_{j-1} Rx(alpha) Tx(a) Tz(d) Rz(q) with dh = (a, d, cos alpha, sin alpha) and (c, s) = (cos q, sin q):
//   Y1 = ca Y + sa Z,  Z1 = -sa Y + ca Z,  o1 = o + a X + d Z1,  X2 = c X + s Y1,  Y2 = -s X + c Y1
// (20 issued instructions instead of building F Rz(q) and a 3x4 compose)
__device__ __forceinline__ void dh_fwd(M34P& T, const float* dh, float c, float s) {
    const float a = dh[0], d = dh[1], ca = dh[2], sa = dh[3];
    const F2 Y1 = fma2(bc(sa), T.r01[2], mul2(bc(ca), T.r01[1]));
    const F2 Z1 = fma2(bc(ca), T.r01[2], mul2(bc(-sa), T.r01[1]));
    const float y1 = fmaf(sa, T.r2[2], ca * T.r2[1]);
    const float z1 = fmaf(ca, T.r2[2], -sa * T.r2[1]);
    T.t01 = fma2(bc(d), Z1, fma2(bc(a), T.r01[0], T.t01));
    T.t2 = fmaf(d, z1, fmaf(a, T.r2[0], T.t2));
    const F2 X = T.r01[0];
    const float x = T.r2[0];
    T.r01[0] = fma2(bc(s), Y1, mul2(bc(c), X));
    T.r01[1] = fma2(bc(c), Y1, mul2(bc(-s), X));
    T.r01[2] = Z1;
    T.r2[0] = fmaf(s, y1, c * x);
    T.r2[1] = fmaf(c, y1, -s * x);
    T.r2[2] = z1;
}
// its inverse: T_{j-1} = T_j Rz(-q) Tz(-d) Tx(-a) Rx(-alpha):
//   X = c X2 - s Y2,  Y1 = s X2 + c Y2,  o = o1 - a X - d Z1,  Y = ca Y1 - sa Z1,  Z = sa Y1 + ca Z1
__device__ __forceinline__ void dh_bwd(M34P& T, const float* dh, float c, float s) {
    const float a = dh[0], d = dh[1], ca = dh[2], sa = dh[3];
    const F2 X = fma2(bc(c), T.r01[0], mul2(bc(-s), T.r01[1]));
    const F2 Y1 = fma2(bc(s), T.r01[0], mul2(bc(c), T.r01[1]));
    const float x = fmaf(c, T.r2[0], -s * T.r2[1]);
    const float y1 = fmaf(s, T.r2[0], c * T.r2[1]);
    T.t01 = fma2(bc(-d), T.r01[2], fma2(bc(-a), X, T.t01));
    T.t2 = fmaf(-d, T.r2[2], fmaf(-a, x, T.t2));
    const F2 Z1 = T.r01[2];
    const float z1 = T.r2[2];
    T.r01[0] = X;
    T.r01[1] = fma2(bc(-sa), Z1, mul2(bc(ca), Y1));
    T.r01[2] = fma2(bc(ca), Z1, mul2(bc(sa), Y1));
    T.r2[0] = x;
    T.r2[1] = fmaf(-sa, z1, ca * y1);
    T.r2[2] = fmaf(ca, z1, sa * y1);
}
__device__ __forceinline__ void xform_p(const M34P& T, float x, float y, float z, float& ox, float& oy, float& oz) {
    const F2 o = fma2(T.r01[0], bc(x), fma2(T.r01[1], bc(y), fma2(T.r01[2], bc(z), T.t01)));
    ox = lo(o);
    oy = hi(o);
    oz = fmaf(T.r2[0], x, fmaf(T.r2[1], y, fmaf(T.r2[2], z, T.t2)));
}

// NS query spheres of a lane, packed in pairs: sphere 2j in the low half of x[j] / y[j] / z[j], 2j + 1 in the high
// half; r = radius + eta.  For odd NS the last high half is a far, radius-0 dummy (never reaches anything).
template <int NS>
struct QSet {
    static constexpr int NP = (NS + 1) / 2;
    F2 x[NP], y[NP], z[NP], r[NP];
    __device__ __forceinline__ float sx(int k) const { return (k & 1) ? hi(x[k >> 1]) : lo(x[k >> 1]); }
    __device__ __forceinline__ float sy(int k) const { return (k & 1) ? hi(y[k >> 1]) : lo(y[k >> 1]); }
    __device__ __forceinline__ float sz(int k) const { return (k & 1) ? hi(z[k >> 1]) : lo(z[k >> 1]); }
    __device__ __forceinline__ float sr(int k) const { return (k & 1) ? hi(r[k >> 1]) : lo(r[k >> 1]); }
    __device__ __forceinline__ void set(int k, float px, float py, float pz, float pr) {   // k compile-time
        if (k & 1) {
            x[k >> 1] = pk(lo(x[k >> 1]), px); y[k >> 1] = pk(lo(y[k >> 1]), py);
            z[k >> 1] = pk(lo(z[k >> 1]), pz); r[k >> 1] = pk(lo(r[k >> 1]), pr);
        } else {
            x[k >> 1] = pk(px, hi(x[k >> 1])); y[k >> 1] = pk(py, hi(y[k >> 1]));
            z[k >> 1] = pk(pz, hi(z[k >> 1])); r[k >> 1] = pk(pr, hi(r[k >> 1]));
        }
    }
    __device__ __forceinline__ void finish() {               // the odd dummy far away
        if (NS & 1) {
            x[NP - 1] = pk(lo(x[NP - 1]), kFar); y[NP - 1] = pk(lo(y[NP - 1]), kFar);
            z[NP - 1] = pk(lo(z[NP - 1]), kFar); r[NP - 1] = pk(lo(r[NP - 1]), 0.f);
        }
    }
};

// does some query sphere reach the sphere (c, rad)?  (d^2 - (r + rad)^2 < 0, the scalar broad-phase test)
template <int NS>
__device__ __forceinline__ bool qset_near(const QSet<NS>& q, float cx, float cy, float cz, float rad) {
    bool near = false;
#pragma unroll
    for (int j = 0; j < QSet<NS>::NP; ++j) {
        const F2 t = reach2(sub2(q.x[j], bc(cx)), sub2(q.y[j], bc(cy)), sub2(q.z[j], bc(cz)), q.r[j], rad);
        near = near || lo(t) < 0.f || hi(t) < 0.f;
    }
    return near;
}

// NS query spheres per lane vs the 8 (padded) spheres of one object instance (shared memory, SoA x[8] y[8] z[8]
// r[8], broadcast to the group).  Fast path: the branch-free test of all NS x 8 pairs (d^2 - (ra+rb)^2 < 0 ?) on
// packed sphere pairs (or, for one query sphere, on packed partner pairs), no square roots, recorded as one bit
// per pair; only if some lane of the warp has an active pair are the exact hinges and gradients of the active
// pairs evaluated.  Returns the hinge sum; if GRAD accumulates dJ/dw_a (x lam) into g and the partner's wrench
// into pw.
template <int NS, class F>
__device__ __forceinline__ void instance_pair_tests(const QSet<NS>& q, const float* X, F&& on) {
    if (!TAMP_PACK_NARROW) {    // scalar: d^2 - R^2 per pair
#pragma unroll
        for (int b = 0; b < TAMP_MAX_OBJ_SPHERES; ++b) {
            const float bx = X[b], by = X[8 + b], bz = X[16 + b], br = X[24 + b];
#pragma unroll
            for (int k = 0; k < NS; ++k) {
                const float dx = q.sx(k) - bx, dy = q.sy(k) - by, dz = q.sz(k) - bz;
                const float R = q.sr(k) + br;
                on(k, b, fmaf(-R, R, fmaf(dx, dx, fmaf(dy, dy, dz * dz))));
            }
        }
    } else if (NS == 1) {      // one query sphere: packed over the partner's sphere pairs (adjacent in the SoA rows)
        const float qx = lo(q.x[0]), qy = lo(q.y[0]), qz = lo(q.z[0]), qr = lo(q.r[0]);
#pragma unroll
        for (int b = 0; b < TAMP_MAX_OBJ_SPHERES; b += 2) {
            const F2 bx = *reinterpret_cast<const F2*>(X + b), by = *reinterpret_cast<const F2*>(X + 8 + b);
            const F2 bz = *reinterpret_cast<const F2*>(X + 16 + b), br = *reinterpret_cast<const F2*>(X + 24 + b);
            const F2 t = reach2(sub2(bx, bc(qx)), sub2(by, bc(qy)), sub2(bz, bc(qz)), br, qr);
            on(0, b, lo(t));
            on(0, b + 1, hi(t));
        }
    } else {
#pragma unroll kNarrowUnroll
        for (int b = 0; b < TAMP_MAX_OBJ_SPHERES; ++b) {
            const F2 bx = bc(X[b]), by = bc(X[8 + b]), bz = bc(X[16 + b]);
            const float br = X[24 + b];
#pragma unroll
            for (int j = 0; j < QSet<NS>::NP; ++j) {
                const F2 t = reach2(sub2(q.x[j], bx), sub2(q.y[j], by), sub2(q.z[j], bz), q.r[j], br);
                on(2 * j, b, lo(t));
                if (2 * j + 1 < NS) on(2 * j + 1, b, hi(t));
            }
        }
    }
}

template <bool GRAD, int NS, class OnWrench>
__device__ __forceinline__ float pairs_vs_instance(const QSet<NS>& q, const float* X, const float4 bound, float lam,
                                                   float (&g)[NS][3], OnWrench&& on_wrench, float smooth) {
    // broad phase: skip the instance unless some query sphere of the warp reaches its bounding sphere
    if (!__any_sync(FULL, qset_near(q, bound.x, bound.y, bound.z, bound.w))) return 0.f;
    // which pairs are active: bit b of act[k] = sign of d^2 - R^2 of pair (k, b) (a -0 or a NaN with the sign bit
    // set only sends an inactive pair to the exact test below, which rejects it again)
    uint32_t act[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) act[k] = 0u;
#if TAMP_FUNNEL_MASK
    // (funnel shift: act[k] = act[k] << 1 | sign(t), one SHF per pair; the pairs arrive in ascending b, so pair b
    // ends at bit 7 - b and the highest set bit is the lowest b)
    instance_pair_tests(q, X, [&](int k, int b, float t) { act[k] = __funnelshift_l(__float_as_uint(t), act[k], 1); });
#else
    instance_pair_tests(q, X, [&](int k, int b, float t) { act[k] |= (__float_as_uint(t) >> 31) << b; });
#endif
    uint32_t any = 0u;
#pragma unroll
    for (int k = 0; k < NS; ++k) any |= act[k];
    if (!__any_sync(FULL, any != 0u)) return 0.f;
    // exact hinges and gradients of the active pairs
    float j = 0.f;
    Wrench pw;
    pw.zero();
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        uint32_t m = act[k];
        while (m) {
#if TAMP_FUNNEL_MASK
            const int hb = 31 - __clz(m);
            m ^= 1u << hb;
            const int b = (TAMP_MAX_OBJ_SPHERES - 1) - hb;
#else
            const int b = __ffs(m) - 1;
            m &= m - 1u;
#endif
            const float4 B = make_float4(X[b], X[8 + b], X[16 + b], X[24 + b]);
            float ux, uy, uz;
            j += sphere_sphere<GRAD>(q.sx(k), q.sy(k), q.sz(k), q.sr(k), B, lam, ux, uy, uz, smooth);
            if (GRAD) {
                g[k][0] -= ux; g[k][1] -= uy; g[k][2] -= uz;
                pw.add_point(B.x, B.y, B.z, ux, uy, uz);
            }
        }
    }
    on_wrench(pw);   // warp-uniform: reduce / store the partner's wrench
    return j;
}

// sphere_obb's exact reject test for a packed pair of spheres with box-frame offsets p and radii r: a sphere reaches
// the box unless s >= r^2, s = ||max(|p| - h, 0)||^2, evaluated as 4 s = ||a + |a|||^2 >= (2r)^2 (a = |p| - h; 2 max(a, 0)
// = a + |a| on the FMA pipe, scaling by 4 exact)
__device__ __forceinline__ void obb_reach_pair(F2 px, F2 py, F2 pz, F2 r, const KObb& B, bool& h0, bool& h1) {
    float qq[2][3];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const float ax = fabsf(h ? hi(px) : lo(px)) - B.h[0];
        const float ay = fabsf(h ? hi(py) : lo(py)) - B.h[1];
        const float az = fabsf(h ? hi(pz) : lo(pz)) - B.h[2];
        qq[h][0] = ax + fabsf(ax);  qq[h][1] = ay + fabsf(ay);  qq[h][2] = az + fabsf(az);
    }
    const F2 qx = pk(qq[0][0], qq[1][0]), qy = pk(qq[0][1], qq[1][1]), qz = pk(qq[0][2], qq[1][2]);
    const F2 s4 = fma2(qx, qx, fma2(qy, qy, mul2(qz, qz)));
    const F2 r2 = add2(r, r);
    const F2 r4 = mul2(r2, r2);
    h0 = !(lo(s4) >= lo(r4));
    h1 = !(hi(s4) >= hi(r4));
}
// Conservative reject test for an axis-aligned box on the sphere centres themselves: per axis
// q = max(w - hi, lo - w, 0) (one FADD2 per corner, a 3-input max) with the corners grown by kCornerSlack, so that
// q <= the exact test's max(|w - c| - h, 0) whatever the fp32 rounding (|coordinates| <= kMaxCoord): a sphere this
// test rejects (||q||^2 >= r^2) is rejected by sphere_obb too; the few it keeps within the slack are evaluated
// exactly (zero hinge).  Results are unchanged.
__device__ __forceinline__ void obb_reach_corner_pair(F2 x, F2 y, F2 z, F2 r, const float4& lo4, const float4& hi4,
                                                      bool& h0, bool& h1) {
    const F2 ux = sub2(x, bc(hi4.x)), vx = sub2(bc(lo4.x), x);
    const F2 uy = sub2(y, bc(hi4.y)), vy = sub2(bc(lo4.y), y);
    const F2 uz = sub2(z, bc(hi4.z)), vz = sub2(bc(lo4.z), z);
    const F2 qx = pk(fmaxf(fmaxf(lo(ux), lo(vx)), 0.f), fmaxf(fmaxf(hi(ux), hi(vx)), 0.f));
    const F2 qy = pk(fmaxf(fmaxf(lo(uy), lo(vy)), 0.f), fmaxf(fmaxf(hi(uy), hi(vy)), 0.f));
    const F2 qz = pk(fmaxf(fmaxf(lo(uz), lo(vz)), 0.f), fmaxf(fmaxf(hi(uz), hi(vz)), 0.f));
    const F2 s = fma2(qx, qx, fma2(qy, qy, mul2(qz, qz)));
    const F2 r2 = mul2(r, r);
    h0 = !(lo(s) >= lo(r2));
    h1 = !(hi(s) >= hi(r2));
}
__device__ __forceinline__ void obb_reach_corner_pair(F2 x, F2 y, F2 z, F2 r, const KObb& B, bool& h0, bool& h1) {
    obb_reach_corner_pair(x, y, z, r, make_float4(B.lo[0], B.lo[1], B.lo[2], 0.f),
                          make_float4(B.hi[0], B.hi[1], B.hi[2], 0.f), h0, h1);
}
// box-frame offsets p = R^T (w - c) of a packed pair of points (aligned boxes: the offsets themselves)
__device__ __forceinline__ void obb_offsets_pair(F2 x, F2 y, F2 z, const KObb& B, F2& px, F2& py, F2& pz) {
    const F2 dx = sub2(x, bc(B.c[0])), dy = sub2(y, bc(B.c[1])), dz = sub2(z, bc(B.c[2]));
    px = dx; py = dy; pz = dz;
    if (!B.aligned) {
        px = fma2(bc(B.R[0]), dx, fma2(bc(B.R[3]), dy, mul2(bc(B.R[6]), dz)));
        py = fma2(bc(B.R[1]), dx, fma2(bc(B.R[4]), dy, mul2(bc(B.R[7]), dz)));
        pz = fma2(bc(B.R[2]), dx, fma2(bc(B.R[5]), dy, mul2(bc(B.R[8]), dz)));
    }
}

// NS query spheres per lane vs one OBB: the exact reject test of every sphere first (packed straight-line code),
// hinge + gradient only for spheres that reach the box, and nothing at all unless some sphere of the warp does.
// Small boxes are first gated by their bounding sphere.  The reject test is sphere_obb's own, s >= r^2 with
// s = ||max(|R^T (w - c)| - h, 0)||^2, evaluated as 4 s = ||a + |a|||^2 >= (2r)^2 (a = |p| - h; scaling by 4 is
// exact) on the FMA pipe; skipped spheres would add exact zeros: results are unchanged.
// fb (optional): the box's fast-path data in shared memory (TAMP_OBB_SMEM: (c, rad), (lo, aligned), (hi, 0)), read
// with three broadcast 16-byte loads instead of indexed constant loads; the exact hinge reads B
template <bool GRAD, int NS, bool ROLLED = false>
__device__ __forceinline__ float spheres_vs_obb(const QSet<NS>& q, const KObb& B, float lam, float (&g)[NS][3],
                                                float smooth, const float4* fb = nullptr) {
    float4 cr, lo4, hi4;
    if (fb) { cr = fb[0]; lo4 = fb[1]; hi4 = fb[2]; }
    else {
        cr = make_float4(B.c[0], B.c[1], B.c[2], B.rad);
        lo4 = make_float4(B.lo[0], B.lo[1], B.lo[2], B.aligned ? 1.f : 0.f);
        hi4 = make_float4(B.hi[0], B.hi[1], B.hi[2], 0.f);
    }
    if (cr.w < kBroadMaxRad) {       // broad phase: bounding sphere of the box (not for boxes larger than the
                                     // arm's reach, e.g. the table, where it would rarely reject)
        if (!__any_sync(FULL, qset_near(q, cr.x, cr.y, cr.z, cr.w))) return 0.f;
    }
    bool hit[NS], any = false;
    if (TAMP_PACK_OBB == 0) {         // scalar: obb_within per sphere
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            hit[k] = obb_within(q.sx(k), q.sy(k), q.sz(k), q.sr(k), B);
            any = any || hit[k];
        }
    } else if (TAMP_BOX_CORNER && TAMP_PACK_OBB == 1 && lo4.w != 0.f) {
#pragma unroll
        for (int j = 0; j < QSet<NS>::NP; ++j) {
            bool h0, h1;
            obb_reach_corner_pair(q.x[j], q.y[j], q.z[j], q.r[j], lo4, hi4, h0, h1);
            hit[2 * j] = h0;
            any = any || h0;
            if (2 * j + 1 < NS) {
                hit[2 * j + 1] = h1;
                any = any || h1;
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < QSet<NS>::NP; ++j) {
            const F2 dx = sub2(q.x[j], bc(B.c[0])), dy = sub2(q.y[j], bc(B.c[1])), dz = sub2(q.z[j], bc(B.c[2]));
            F2 px = dx, py = dy, pz = dz;
            if (!B.aligned) {            // p = R^T (w - c)
                px = fma2(bc(B.R[0]), dx, fma2(bc(B.R[3]), dy, mul2(bc(B.R[6]), dz)));
                py = fma2(bc(B.R[1]), dx, fma2(bc(B.R[4]), dy, mul2(bc(B.R[7]), dz)));
                pz = fma2(bc(B.R[2]), dx, fma2(bc(B.R[5]), dy, mul2(bc(B.R[8]), dz)));
            }
            if (TAMP_PACK_OBB == 1) {   // 2 max(a, 0) = a + |a| on the FMA pipe; 4 s >= (2r)^2 (scaling by 4 exact)
                bool h0, h1;
                obb_reach_pair(px, py, pz, q.r[j], B, h0, h1);
                hit[2 * j] = h0;
                any = any || h0;
                if (2 * j + 1 < NS) {
                    hit[2 * j + 1] = h1;
                    any = any || h1;
                }
            } else {                    // obb_within's own formula on the packed offsets
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (2 * j + h >= NS) continue;
                    const float r = h ? hi(q.r[j]) : lo(q.r[j]);
                    const float ax = fabsf(h ? hi(px) : lo(px)) - B.h[0];
                    const float ay = fabsf(h ? hi(py) : lo(py)) - B.h[1];
                    const float az = fabsf(h ? hi(pz) : lo(pz)) - B.h[2];
                    const float qx = fmaxf(ax, 0.f), qy = fmaxf(ay, 0.f), qz = fmaxf(az, 0.f);
                    const bool out = fmaxf(ax, fmaxf(ay, az)) > 0.f && fmaf(qx, qx, fmaf(qy, qy, qz * qz)) >= r * r;
                    hit[2 * j + h] = !out;
                    any = any || !out;
                }
            }
        }
    }
    float j = 0.f;
    if (__any_sync(FULL, any)) {
        if (ROLLED) {
            // one rolled copy of the exact hinge over the hit bits in ascending sphere order (the same sums and
            // the same fused accumulations as one unrolled block per sphere): operands and the sphere's gradient
            // accumulator selected from registers -- a smaller kernel body (instruction cache)
            unsigned hm = 0;
#pragma unroll
            for (int k = 0; k < NS; ++k) hm |= hit[k] ? 1u << k : 0u;
#pragma unroll 1
            while (hm) {
                const int k = __ffs(hm) - 1;
                hm &= hm - 1;
                float x = q.sx(0), y = q.sy(0), z = q.sz(0), r = q.sr(0);
                float gx = g[0][0], gy = g[0][1], gz = g[0][2];
#pragma unroll
                for (int u = 1; u < NS; ++u)
                    if (k == u) { x = q.sx(u); y = q.sy(u); z = q.sz(u); r = q.sr(u); gx = g[u][0]; gy = g[u][1]; gz = g[u][2]; }
                j += sphere_obb<GRAD>(x, y, z, r, B, lam, gx, gy, gz, smooth);
#pragma unroll
                for (int u = 0; u < NS; ++u)
                    if (k == u) { g[u][0] = gx; g[u][1] = gy; g[u][2] = gz; }
            }
        } else {
#pragma unroll
            for (int k = 0; k < NS; ++k)
                if (hit[k]) j += sphere_obb<GRAD>(q.sx(k), q.sy(k), q.sz(k), q.sr(k), B, lam, g[k][0], g[k][1], g[k][2], smooth);
        }
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

// Value of a term that is a sum of per-lane parts (collision hinges, containment): reduced over the group for
// the check / eval, whose per-term values and J must be exact.  The optimisation step needs J only for its
// finiteness test (the gradient is assembled separately), and the group ballot of that test sees a non-finite
// part on any lane, so it keeps the parts lane-local and skips the shuffle chain.
template <int MODE, int W>
__device__ __forceinline__ float term_sum(float v) {
    return MODE == MODE_OPT ? v : gsum<W>(v);
}

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
// share the instruction cache.  0 = off (warp-level only), 1 = one block barrier per step, after the FK loop
// (every other phase boundary only needs its particle group, i.e. __syncwarp; measured best: barriers at
// every phase boundary cost 3 %), 2 = also after every FK instance.
// SMOOTH: CHOMP-smooth collision cost (compile-time so that the hinge kernels carry no extra state)
// MAXT: launch bound -- 768 (<= 80 registers: many resident warps for multi-wave launches) or 512 (<= 128
// registers, no spills: single-wave launches of <= 512-thread blocks and the 16-lane mapping; +7 % on config 2,
// +24 % on config 4)
template <int MODE, int LPF, int HP, int BSYNC, bool SMOOTH, int MAXT>
__global__ void __launch_bounds__(MAXT, 1) k_particle(const __grid_constant__ KProgram P, const KArgs A) {
    constexpr bool GRAD = MODE != MODE_CHECK;
    const float smooth = SMOOTH ? P.smooth : 0.f;
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
    __shared__ __align__(16) float s_rsoa[kGroup][4 * TAMP_MAX_SPHERES_PER_LINK];   // the same, SoA x[4] y[4] z[4] r[4]
    __shared__ uint32_t s_selfmask[kGroup * TAMP_MAX_SPHERES_PER_LINK];
    // boxes' fast-path data (broad phase and corner reject test): (c, rad), (lo, aligned), (hi, 0) per box
    __shared__ float4 s_obb[TAMP_OBB_SMEM ? TAMP_MAX_OBB : 1][3];

    const int gl = threadIdx.x & (GS - 1);          // lane within the particle group
    const int ll = gl & (LPF - 1);                  // lane within the FK segment
    const int half = gl / LPF;                      // HP = 2: which FK instance of the pair
    const int grp = threadIdx.x / GS;
    const int64_t pid = (int64_t)blockIdx.x * (blockDim.x / GS) + grp;
    const bool active = pid < A.n;
    const int64_t p = active ? pid : (A.n - 1);
    // dynamic shared memory: [constant instances, shared by the block | per-particle areas of A.stride floats]
    float* const cinst = reinterpret_cast<float*>(smem4);
    float* S = cinst + A.const_floats + (size_t)grp * A.stride;
    float* xs = S;
    float* gs = S + A.off_g;
    float* const minst = S + A.off_inst;
    float* gT = S + A.off_gT;
    float* gTi = S + A.off_gTi;
    // an object instance's block of kInstFloats floats: [pose rows 3x4 | world bounding sphere | 8 world sphere
    // centres (float4) | wrench (movable only)]; constant instances live once per block, movable ones per particle
    auto inst = [&](int i) -> float* {
        const KInst& I = P.inst[i];
        TAMP_DCHECK(i >= 0 && i < P.n_inst && I.slot >= 0);
        TAMP_DCHECK(I.xoff >= 0 ? A.off_inst + kInstFloats * (I.slot + 1) <= A.stride
                                : kInstFloats * (I.slot + 1) <= A.const_floats);
        return (I.xoff >= 0 ? minst : cinst) + kInstFloats * I.slot;
    };
    TAMP_DCHECK(A.const_floats + (grp + 1) * A.stride <= A.smem_floats);
    TAMP_DCHECK(A.fk_off + P.n_fk * (int)(sizeof(KFk) / 4) <= A.const_floats);
    TAMP_DCHECK(A.pw_off + A.n_pw <= A.const_floats);
    TAMP_DCHECK(A.off_g + P.D <= A.stride && A.off_gT + 12 * P.n_grasp <= A.stride);
    TAMP_DCHECK(A.off_gTi < 0 || A.off_gTi + 12 * P.n_grasp <= A.stride);
    TAMP_DCHECK(!P.has_self || A.off_rsw + 4 * HP * kGroup * TAMP_MAX_SPHERES_PER_LINK <= A.stride);
    auto ipose = [&](int i) -> float* { return inst(i); };
    auto iwr = [&](int i) -> float* { return inst(i) + 48; };
    const int D = P.D;
    auto phase_sync = [&]() {
        if (BSYNC > 0) __syncthreads(); else __syncwarp();
    };

    for (int i = threadIdx.x; i < TAMP_MAX_OBJECTS * TAMP_MAX_OBJ_SPHERES; i += blockDim.x) {
        const int o = i / TAMP_MAX_OBJ_SPHERES, k = i % TAMP_MAX_OBJ_SPHERES;
        s_osph[o][k] = make_float4(P.osph[o][k][0], P.osph[o][k][1], P.osph[o][k][2], P.osph[o][k][3]);
    }
    if (MODE == MODE_CHECK || (MODE == MODE_OPT && A.check_after))
        for (int i = threadIdx.x; i < P.n_terms + 2; i += blockDim.x) s_counts[i] = 0;
    // the configurations' descriptors, once per block; each FK instance takes a register copy of its descriptor
    // from shared memory (FKS) instead of indexed constant loads plus their address computation at every use of a
    // field (the compiler re-derived them rather than keep registers): config 4 7.76 -> 7.18 ms, config 2 -2 %,
    // config 3 -0.5 %
    constexpr bool FKS = TAMP_FK_SMEM && MAXT <= TAMP_FK_SMEM_MAXT;
    KFk* const s_fk = reinterpret_cast<KFk*>(cinst + A.fk_off);
    // partner reference k as an offset word (>= 0: movable instance, from the particle's area; < 0: constant, ~offset
    // from the block's constant area): one shared load per partner instead of the instance lookup
    constexpr bool PTAB = TAMP_PARTNER_TABLE && MAXT <= 512;
    int* const s_pw = reinterpret_cast<int*>(cinst + A.pw_off);
    if (PTAB)
        for (int k = threadIdx.x; k < A.n_pw; k += blockDim.x) {
            const KInst& I = P.inst[P.partners[k]];
            s_pw[k] = I.xoff >= 0 ? A.off_inst + kInstFloats * I.slot : ~(kInstFloats * I.slot);
        }
    if (FKS)
        for (int i = threadIdx.x; i < P.n_fk; i += blockDim.x) s_fk[i] = P.fk[i];
    if (TAMP_OBB_SMEM && threadIdx.x < P.n_obb) {
        const KObb& B = P.obb[threadIdx.x];
        s_obb[threadIdx.x][0] = make_float4(B.c[0], B.c[1], B.c[2], B.rad);
        s_obb[threadIdx.x][1] = make_float4(B.lo[0], B.lo[1], B.lo[2], B.aligned ? 1.f : 0.f);
        s_obb[threadIdx.x][2] = make_float4(B.hi[0], B.hi[1], B.hi[2], 0.f);
    }
    if (threadIdx.x < kGroup * 3) {
        const int l = threadIdx.x / 3, r = threadIdx.x % 3;
        s_F[l][r] = make_float4(P.F[l][4 * r], P.F[l][4 * r + 1], P.F[l][4 * r + 2], P.F[l][4 * r + 3]);
    }
    if (threadIdx.x < kGroup * TAMP_MAX_SPHERES_PER_LINK) {
        const int l = threadIdx.x / TAMP_MAX_SPHERES_PER_LINK, k = threadIdx.x % TAMP_MAX_SPHERES_PER_LINK;
        s_rsph[l][k] = make_float4(P.rsph[l][k][0], P.rsph[l][k][1], P.rsph[l][k][2], P.rsph[l][k][3]);
#pragma unroll
        for (int c = 0; c < 4; ++c) s_rsoa[l][TAMP_MAX_SPHERES_PER_LINK * c + k] = P.rsph[l][k][c];
        s_selfmask[threadIdx.x] = P.self_mask[threadIdx.x];
    }
    float4* rsw = reinterpret_cast<float4*>(S + A.off_rsw) + (HP > 1 ? half : 0) * (kGroup * TAMP_MAX_SPHERES_PER_LINK);
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
#pragma unroll 4
    for (int d = gl; d < D; d += GS) xs[d] = xg[d];
    const float* gg = A.grasp + (p * P.n_grasp) * 12;
#pragma unroll 4
    for (int i = gl; i < P.n_grasp * 12; i += GS) gT[i] = gg[i];
    bool invalid = A.invalid[p] != 0;
    // constant object instances (bold p0 constants): pose and world spheres, once per block
    for (int i = 0; i < P.n_inst; ++i) {
        const KInst& I = P.inst[i];
        if (I.xoff >= 0) continue;
        float sy, cy;
        fsincos(I.pose[3], &sy, &cy);
        float* ip = cinst + kInstFloats * I.slot;
        const float px = I.pose[0], py = I.pose[1], pz = I.pose[2];
        for (int k = threadIdx.x; k <= TAMP_MAX_OBJ_SPHERES; k += blockDim.x) {
            if (k == TAMP_MAX_OBJ_SPHERES) {
                ip[0] = cy; ip[1] = -sy; ip[2] = 0.f; ip[3] = px;
                ip[4] = sy; ip[5] = cy; ip[6] = 0.f; ip[7] = py;
                ip[8] = 0.f; ip[9] = 0.f; ip[10] = 1.f; ip[11] = pz;
                const float* ob = P.obound[I.obj];
                ip[12] = fmaf(cy, ob[0], fmaf(-sy, ob[1], px));
                ip[13] = fmaf(sy, ob[0], fmaf(cy, ob[1], py));
                ip[14] = pz + ob[2];
                ip[15] = ob[3];
            } else {                                  // spheres SoA: x[8] y[8] z[8] r[8]
                const float* c = P.osph[I.obj][k];
                const bool in = k < P.osph_n[I.obj];
                ip[16 + k] = in ? fmaf(cy, c[0], fmaf(-sy, c[1], px)) : kFar;
                ip[24 + k] = in ? fmaf(sy, c[0], fmaf(cy, c[1], py)) : kFar;
                ip[32 + k] = in ? pz + c[2] : kFar;
                ip[40 + k] = in ? c[3] : 0.f;
            }
        }
    }
    __syncthreads();
    if (A.off_gTi >= 0) {   // inverse grasps (held objects at knots): one grasp per lane of the group
        for (int k = gl; k < P.n_grasp; k += GS) {
            M34 g, gi;
            load_m34(g, gT + 12 * k);
            inv_m34(g, gi);
            float* o = gTi + 12 * k;
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                o[4 * i] = gi.r[3 * i]; o[4 * i + 1] = gi.r[3 * i + 1]; o[4 * i + 2] = gi.r[3 * i + 2];
                o[4 * i + 3] = gi.t[i];
            }
        }
    }
    __syncwarp();

    const int n_iter = (MODE == MODE_OPT) ? A.n_steps : 1;
    // one optimisation / check / eval iteration; M = MODE, or MODE_CHECK for the check fused after the last step
    auto iteration = [&](auto mtag, const int it) {
        constexpr int M = decltype(mtag)::value;
        constexpr bool G = M != MODE_CHECK;
        TermSink<M> sink;
        float soft = 0.f;

        // ---- phase A: movable object instances (poses, world sphere centres), zero accumulators ----
        for (int i = 0; i < P.n_inst; ++i) {
            const KInst& I = P.inst[i];
            if (I.xoff < 0) continue;      // constant instances: set up once per block (prologue)
            TAMP_DCHECK(I.xoff + 4 <= D);
            const float px = xs[I.xoff], py = xs[I.xoff + 1], pz = xs[I.xoff + 2], yaw = xs[I.xoff + 3];
            float sy, cy;
            fsincos(yaw, &sy, &cy);
            float* ip = minst + kInstFloats * I.slot;   // [R row0 | t0, R row1 | t1, R row2 | t2, bounding sphere]
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
                const bool in = k < P.osph_n[I.obj];     // spheres SoA: x[8] y[8] z[8] r[8]
                ip[16 + k] = in ? fmaf(cy, c.x, fmaf(-sy, c.y, px)) : kFar;
                ip[24 + k] = in ? fmaf(sy, c.x, fmaf(cy, c.y, py)) : kFar;
                ip[32 + k] = in ? pz + c.z : kFar;
                ip[40 + k] = in ? c.w : 0.f;
            }
            if (G)
                for (int c = gl; c < 6; c += GS) ip[48 + c] = 0.f;
        }
        if (G) for (int d = gl; d < D; d += GS) gs[d] = 0.f;
        __syncwarp();

        // ---- phase B: robot configurations (Pick/Place confs, knots) ----
        // HP = 2: the two halves process the two FK instances of a pair of identical structure concurrently
        // (the compiler pairs them; an unmatched instance is paired with a ghost copy whose results are
        // discarded), so control flow stays warp-uniform.  HP = 1: ghosts are skipped.
        TermSink<M> sinkB;                  // this half's share of the phase-B terms
        for (int f0 = 0; f0 < P.n_fk; f0 += HP) {
            KFk Kc;
            if (!FKS || TAMP_FK_COPY) Kc = FKS ? s_fk[f0 + (HP > 1 ? half : 0)] : P.fk[f0 + (HP > 1 ? half : 0)];
            const KFk& K = FKS && !TAMP_FK_COPY ? s_fk[f0 + (HP > 1 ? half : 0)] : Kc;
            const bool real = !K.ghost;
            TAMP_DCHECK(f0 + HP <= TAMP_MAX_FK && K.xoff >= 0 && K.xoff + TAMP_NJ <= D);
            TAMP_DCHECK(K.part_begin >= 0 && K.part_begin + K.part_count <= kMaxPartners);
            TAMP_DCHECK(K.kin_grasp < P.n_grasp && K.held_grasp < P.n_grasp);
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
            // (the scan's partial products keep rows 0-1 packed: FFMA2 composes, the scalar composes' values)
            M34P Sp = pack_m34(Al[0]);
            if (LPL == 2) Sp = compose_p(Sp, Al[LPL - 1]);
#pragma unroll
            for (int d = 1; d < LPF; d <<= 1) {
                const M34P U = shfl_up_m34p(Sp, d, LPF);
                if (ll >= d) Sp = compose_p(U, unpack_m34(Sp));
            }
            M34 T[LPL];                       // my link frames (world)
            if (LPL == 1) {
                T[0] = unpack_m34(Sp);
            } else {
                const M34P E = shfl_up_m34p(Sp, 1, LPF);   // product of all earlier lanes' transforms
                T[0] = ll == 0 ? Al[0] : unpack_m34(compose_p(E, Al[0]));
                T[LPL - 1] = unpack_m34(Sp);
            }
            const float lam_cf = K.term_cf >= 0 ? P.term_lam[K.term_cf] : 0.f;
            // my links' spheres in the world, transformed in packed pairs (w = T c, the xform order)
            QSet<NS> rs;
            float gw[NS][3];
#pragma unroll
            for (int u = 0; u < LPL; ++u) {
                const float* cs = s_rsoa[ll * LPL + u];          // x[4] y[4] z[4] r[4] in the link frame
#pragma unroll
                for (int kp = 0; kp < TAMP_MAX_SPHERES_PER_LINK / 2; ++kp) {
                    const int j = u * (TAMP_MAX_SPHERES_PER_LINK / 2) + kp;
                    if (!TAMP_PACK_XFORM) {
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            float wx, wy, wz;
                            xform(T[u], cs[2 * kp + h], cs[4 + 2 * kp + h], cs[8 + 2 * kp + h], wx, wy, wz);
                            rs.set(2 * j + h, wx, wy, wz, cs[12 + 2 * kp + h] + P.eta);
                        }
                        continue;
                    }
                    const F2 cx = *reinterpret_cast<const F2*>(cs + 2 * kp);
                    const F2 cy = *reinterpret_cast<const F2*>(cs + 4 + 2 * kp);
                    const F2 cz = *reinterpret_cast<const F2*>(cs + 8 + 2 * kp);
                    const F2 cr = *reinterpret_cast<const F2*>(cs + 12 + 2 * kp);
                    rs.x[j] = fma2(bc(T[u].r[0]), cx, fma2(bc(T[u].r[1]), cy, fma2(bc(T[u].r[2]), cz, bc(T[u].t[0]))));
                    rs.y[j] = fma2(bc(T[u].r[3]), cx, fma2(bc(T[u].r[4]), cy, fma2(bc(T[u].r[5]), cz, bc(T[u].t[1]))));
                    rs.z[j] = fma2(bc(T[u].r[6]), cx, fma2(bc(T[u].r[7]), cy, fma2(bc(T[u].r[8]), cz, bc(T[u].t[2]))));
                    rs.r[j] = add2(cr, bc(P.eta));
                }
                if (nsph[u] < TAMP_MAX_SPHERES_PER_LINK) {         // absent sphere slots: far away
#pragma unroll
                    for (int k = 0; k < TAMP_MAX_SPHERES_PER_LINK; ++k) {
                        const int s2 = u * TAMP_MAX_SPHERES_PER_LINK + k;
                        if (k >= nsph[u]) rs.set(s2, kFar, kFar, kFar, rs.sr(s2));
                    }
                }
            }
            rs.finish();
#pragma unroll
            for (int s2 = 0; s2 < NS; ++s2) gw[s2][0] = gw[s2][1] = gw[s2][2] = 0.f;
            float jcf = 0.f;
            if (K.term_cf >= 0) {
                // robot spheres vs OBBs (constant cache)
                for (int b = 0; b < P.n_obb; ++b)
                    if ((K.obb_mask >> b) & 1) jcf += spheres_vs_obb<G, NS, TAMP_ROLLED_HITS && (HP > 1)>(rs, P.obb[b], lam_cf, gw, smooth, TAMP_OBB_SMEM ? s_obb[b] : nullptr);
                // robot spheres vs movable objects' spheres (shared memory)
                for (int pi = 0; pi < K.part_count; ++pi) {
                    float* ip;
                    bool mov;
                    if (PTAB) {
                        TAMP_DCHECK(K.part_begin + pi < A.n_pw);
                        const int w = s_pw[K.part_begin + pi];
                        ip = w >= 0 ? S + w : cinst + ~w;
                        mov = w >= 0;
                    } else {
                        const int ii = P.partners[K.part_begin + pi];
                        ip = inst(ii);
                        mov = P.inst[ii].xoff >= 0;
                    }
                    jcf += pairs_vs_instance<G, NS>(rs, ip + 16, *reinterpret_cast<const float4*>(ip + 12), lam_cf, gw,
                        [&](Wrench& pw) { flush_partner_b<G, HP, LPF>(pw, mov, ip + 48, ll, half, real); }, smooth);
                }
            }
            // robot self-collision: every lane tests its own spheres against the configuration's
            // robot spheres (centres shared through shared memory) in packed pairs -- d^2 - (r_a + r_b)^2 as the
            // exact reject test, its sign bits ANDed with the pair mask -- and evaluates the exact hinges of the
            // active pairs, keeping only its own spheres' gradient; each pair's hinge is counted once, by the lower
            // sphere id
            static_assert(kGroup * TAMP_MAX_SPHERES_PER_LINK == 32, "self-pair masks: one bit per robot sphere");
            if (K.term_self >= 0) {
#pragma unroll
                for (int s = 0; s < NS; ++s)
                    rsw[ll * NS + s] = make_float4(rs.sx(s), rs.sy(s), rs.sz(s), rs.sr(s) - P.eta);
                __syncwarp();
                float js = 0.f;
                const float lam_self = P.term_lam[K.term_self];
                uint32_t sact[NS];
#pragma unroll
                for (int s = 0; s < NS; ++s) sact[s] = 0u;
#pragma unroll 4
                for (int t = 0; t < kGroup * TAMP_MAX_SPHERES_PER_LINK; ++t) {
                    const float4 B = rsw[t];
#pragma unroll
                    for (int j = 0; j < QSet<NS>::NP; ++j) {
                        const F2 tt = reach2(sub2(rs.x[j], bc(B.x)), sub2(rs.y[j], bc(B.y)), sub2(rs.z[j], bc(B.z)),
                                             rs.r[j], B.w);
#if TAMP_FUNNEL_MASK                // (pair t ends at bit 31 - t: the pair mask is bit-reversed to match)
                        sact[2 * j] = __funnelshift_l(__float_as_uint(lo(tt)), sact[2 * j], 1);
                        if (2 * j + 1 < NS) sact[2 * j + 1] = __funnelshift_l(__float_as_uint(hi(tt)), sact[2 * j + 1], 1);
#else
                        sact[2 * j] |= (__float_as_uint(lo(tt)) >> 31) << t;
                        if (2 * j + 1 < NS) sact[2 * j + 1] |= (__float_as_uint(hi(tt)) >> 31) << t;
#endif
                    }
                }
#pragma unroll
                for (int s = 0; s < NS; ++s) {
                    const int sid = ll * NS + s;
#if TAMP_FUNNEL_MASK
                    uint32_t m = __brev(s_selfmask[sid]) & sact[s];
                    while (m) {
                        const int hb = 31 - __clz(m);
                        m ^= 1u << hb;
                        const int t = 31 - hb;
#else
                    uint32_t m = s_selfmask[sid] & sact[s];
                    while (m) {
                        const int t = __ffs(m) - 1;
                        m &= m - 1u;
#endif
                        float ux, uy, uz;
                        const float pen = sphere_sphere<G>(rs.sx(s), rs.sy(s), rs.sz(s), rs.sr(s), rsw[t], lam_self, ux, uy,
                                                              uz, smooth);
                        if (sid < t) js += pen;
                        if (G) { gw[s][0] -= ux; gw[s][1] -= uy; gw[s][2] -= uz; }
                    }
                }
                finish_term<M>(P, A, sinkB, K.term_self, term_sum<M, LPF>(js), ll, active, p, s_counts, real);
                __syncwarp();
            }
            Wrench Wl[LPL];                   // wrench (about the world origin) on each of my links
#pragma unroll
            for (int u = 0; u < LPL; ++u) {
                Wl[u].zero();
                if (G) {
#pragma unroll
                    for (int k = 0; k < TAMP_MAX_SPHERES_PER_LINK; ++k) {
                        const int s = u * TAMP_MAX_SPHERES_PER_LINK + k;
                        Wl[u].add_point(rs.sx(s), rs.sy(s), rs.sz(s), gw[s][0], gw[s][1], gw[s][2]);
                    }
                }
            }
            // tool frame to every lane of the segment
            const M34 Tee = shfl_m34(T[LPL - 1], LPF - 1, LPF);
            // held object at a MoveHold knot: attached spheres T_ee T(g)^-1 c (CFreeTrajHold)
            if (K.held_grasp >= 0 && K.term_cf >= 0) {
                M34 Gi, Tobj;
                load_m34(Gi, gTi + 12 * K.held_grasp);
                Tobj = compose(Tee, Gi);
                const int ho = K.held_obj;
                QSet<NH> hq;
                float gh[NH][3];
#pragma unroll
                for (int v = 0; v < NH; ++v) {
                    const int k = ll + LPF * v;
                    const float4 c = s_osph[ho][k];
                    float hx, hy, hz;
                    xform(Tobj, c.x, c.y, c.z, hx, hy, hz);
                    if (k >= P.osph_n[ho]) hx = hy = hz = kFar;
                    hq.set(v, hx, hy, hz, c.w + P.eta);
                    gh[v][0] = gh[v][1] = gh[v][2] = 0.f;
                }
                hq.finish();
                for (int b = 0; b < P.n_obb; ++b)
                    if ((K.obb_mask >> b) & 1) jcf += spheres_vs_obb<G, NH, TAMP_ROLLED_HITS && (HP > 1)>(hq, P.obb[b], lam_cf, gh, smooth, TAMP_OBB_SMEM ? s_obb[b] : nullptr);
                for (int pi = 0; pi < K.part_count; ++pi) {
                    float* ip;
                    bool mov;
                    if (PTAB) {
                        TAMP_DCHECK(K.part_begin + pi < A.n_pw);
                        const int w = s_pw[K.part_begin + pi];
                        ip = w >= 0 ? S + w : cinst + ~w;
                        mov = w >= 0;
                    } else {
                        const int ii = P.partners[K.part_begin + pi];
                        ip = inst(ii);
                        mov = P.inst[ii].xoff >= 0;
                    }
                    jcf += pairs_vs_instance<G, NH>(hq, ip + 16, *reinterpret_cast<const float4*>(ip + 12), lam_cf, gh,
                        [&](Wrench& pw) { flush_partner_b<G, HP, LPF>(pw, mov, ip + 48, ll, half, real); }, smooth);
                }
                if (G) {   // held-object wrench acts on the tool link (last lane of the segment)
                    Wrench hw;
                    hw.zero();
#pragma unroll
                    for (int v = 0; v < NH; ++v) hw.add_point(hq.sx(v), hq.sy(v), hq.sz(v), gh[v][0], gh[v][1], gh[v][2]);
                    hw.template group_sum<LPF>();
                    if (ll == LPF - 1) {
#pragma unroll
                        for (int i = 0; i < 3; ++i) { Wl[LPL - 1].f[i] += hw.f[i]; Wl[LPL - 1].m[i] += hw.m[i]; }
                    }
                }
            }
            if (K.term_cf >= 0)
                finish_term<M>(P, A, sinkB, K.term_cf, term_sum<M, LPF>(jcf), ll, active, p, s_counts, real);

            // Kin(q, o, g, p): FK(q) = T(p) T(g); residuals on every lane of the segment
            if (K.term_kp >= 0 || K.term_kr >= 0) {
                M34 Tg;
                load_m34(Tg, gT + 12 * K.kin_grasp);
                const M34 Ts = compose_rz(ipose(K.kin_inst), Tg);
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
                if (K.term_kp >= 0) finish_term<M>(P, A, sinkB, K.term_kp, epos, ll, active, p, s_counts, real);
                if (K.term_kr >= 0) finish_term<M>(P, A, sinkB, K.term_kr, erot, ll, active, p, s_counts, real);
                if (G) {
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
                        if (half == h && ll == 0 && real && movable) add_wrench(iwr(K.kin_inst), tw);
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
                // inside the limits (always after the projection, L11) every part is 0: skip the shuffle chain
                jl = __any_sync(FULL, e2 > 0.f) ? sqrtf(gsum<LPF>(e2)) : 0.f;
                finish_term<M>(P, A, sinkB, K.term_jl, jl, ll, active, p, s_counts, real);
            }
            if (G) {
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
            if (BSYNC == 2) __syncthreads();
        }
        if (BSYNC == 1) phase_sync();   // all warps leave the FK loop before phase C
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
            // (TAMP_PLACE_PIN: the Place descriptor's fields pinned in registers by opaque copies -- else re-derived
            // from the constant bank at every use)
            KPlace Qc = P.place[pl];
            if (TAMP_PLACE_PIN) {
                Qc.inst = (int16_t)opaque_int(Qc.inst); Qc.term_ss = (int16_t)opaque_int(Qc.term_ss);
                Qc.term_sc = (int16_t)opaque_int(Qc.term_sc); Qc.term_cp = (int16_t)opaque_int(Qc.term_cp);
                Qc.term_pc = (int16_t)opaque_int(Qc.term_pc); Qc.surface = (int16_t)opaque_int(Qc.surface);
                Qc.part_begin = (int16_t)opaque_int(Qc.part_begin); Qc.part_count = (int16_t)opaque_int(Qc.part_count);
                Qc.obb_mask = (uint16_t)opaque_int(Qc.obb_mask);
            }
            const KPlace& Q = TAMP_PLACE_PIN ? Qc : P.place[pl];
            const int ii = Q.inst;
            const KInst& I = P.inst[ii];
            const KSurface& Sf = P.surf[Q.surface];
            const float pz = xs[I.xoff + 2];
            Wrench own;
            own.zero();
            // support: |z_bottom - z_top|  (L6; object frame origin at its bottom, L15); for a press the
            // pressing object's bottom at the button-face height (R8)
            {
                const float e = fabsf(pz - Sf.frame[2]);
                finish_term<M>(P, A, sink, Q.term_ss, e, gl, active, p, s_counts);
                if (G && gl == 0 && e > 0.f) {
                    const float g = P.term_lam[Q.term_ss] * (pz > Sf.frame[2] ? 1.f : -1.f);
                    own.add_point(xs[I.xoff], xs[I.xoff + 1], pz, 0.f, 0.f, g);
                }
            }
            const int no = P.osph_n[I.obj];
            float* const oip = minst + kInstFloats * I.slot;      // the placed object's instance (movable)
            float wq[NSO][3], rq[NSO], gq[NSO][3];
#pragma unroll
            for (int u = 0; u < NSO; ++u) {
                const int k = gl + GS * u;
                const bool in = k < TAMP_MAX_OBJ_SPHERES;           // padded slots: far
                wq[u][0] = in ? oip[16 + k] : kFar;
                wq[u][1] = in ? oip[24 + k] : kFar;
                wq[u][2] = in ? oip[32 + k] : kFar;
                rq[u] = in ? oip[40 + k] : 0.f;
                gq[u][0] = gq[u][1] = gq[u][2] = 0.f;
            }
            // containment: sum over spheres of dist_from_bounds(xy in surface frame, lo + r, hi - r)
            if (Q.term_sc >= 0) {
                const float sy = Sf.sy, cy = Sf.cy;
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
                    if (G && eu > 0.f) {
                        const float k = P.term_lam[Q.term_sc] / eu;
                        const float glx = (lx > hix ? ex : (lx < lox ? -ex : 0.f)) * k;
                        const float gly = (ly > hiy ? ey : (ly < loy ? -ey : 0.f)) * k;
                        gq[u][0] += fmaf(cy, glx, -sy * gly);
                        gq[u][1] += fmaf(sy, glx, cy * gly);
                    }
                }
                finish_term<M>(P, A, sink, Q.term_sc, term_sum<M, GS>(e), gl, active, p, s_counts);
            }
            // press contact (ValidPress / ValidStickPress, R8): min over the object's spheres of
            // dist_from_bounds(xy in the face frame, lo, hi); the subgradient goes to the arg-min sphere
            // (lowest index on ties)
            if (Q.term_pc >= 0) {
                const float sy = Sf.sy, cy = Sf.cy;
                float emin = kFar, glx_min = 0.f, gly_min = 0.f;
                int kmin = TAMP_MAX_OBJ_SPHERES;
#pragma unroll
                for (int u = 0; u < NSO; ++u) {
                    if (gl + GS * u >= no) continue;
                    const float rx = wq[u][0] - Sf.frame[0], ry = wq[u][1] - Sf.frame[1];
                    const float lx = fmaf(cy, rx, sy * ry), ly = fmaf(-sy, rx, cy * ry);
                    const float ex = fmaxf(fmaxf(Sf.lo[0] - lx, lx - Sf.hi[0]), 0.f);
                    const float ey = fmaxf(fmaxf(Sf.lo[1] - ly, ly - Sf.hi[1]), 0.f);
                    const float eu = sqrtf(fmaf(ex, ex, ey * ey));
                    if (eu < emin) {
                        emin = eu;
                        kmin = gl + GS * u;
                        glx_min = eu > 0.f ? (lx > Sf.hi[0] ? ex : (lx < Sf.lo[0] ? -ex : 0.f)) / eu : 0.f;
                        gly_min = eu > 0.f ? (ly > Sf.hi[1] ? ey : (ly < Sf.lo[1] ? -ey : 0.f)) / eu : 0.f;
                    }
                }
#pragma unroll
                for (int o = GS / 2; o > 0; o >>= 1) {
                    const float e2 = __shfl_xor_sync(FULL, emin, o, GS);
                    const int k2 = __shfl_xor_sync(FULL, kmin, o, GS);
                    if (e2 < emin || (e2 == emin && k2 < kmin)) { emin = e2; kmin = k2; }
                }
                finish_term<M>(P, A, sink, Q.term_pc, emin, gl, active, p, s_counts);
                if (G && emin > 0.f) {
                    const float lam = P.term_lam[Q.term_pc];
#pragma unroll
                    for (int u = 0; u < NSO; ++u)
                        if (gl + GS * u == kmin) {
                            gq[u][0] += lam * fmaf(cy, glx_min, -sy * gly_min);
                            gq[u][1] += lam * fmaf(sy, glx_min, cy * gly_min);
                        }
                }
            }
            // CFreePlace: placed-object spheres vs OBBs (support excluded) and other objects
            if (Q.term_cp >= 0) {
                const float lam_cp = P.term_lam[Q.term_cp];
                QSet<NSO> qe;
#pragma unroll
                for (int u = 0; u < NSO; ++u) qe.set(u, wq[u][0], wq[u][1], wq[u][2], rq[u] + P.eta);
                qe.finish();
                float jcp = 0.f;
                for (int b = 0; b < P.n_obb; ++b)
                    if ((Q.obb_mask >> b) & 1) jcp += spheres_vs_obb<G, NSO, TAMP_ROLLED_HITS && (HP > 1)>(qe, P.obb[b], lam_cp, gq, smooth, TAMP_OBB_SMEM ? s_obb[b] : nullptr);
                for (int pi = 0; pi < Q.part_count; ++pi) {
                    float* jp;
                    bool mov;
                    if (PTAB) {
                        TAMP_DCHECK(Q.part_begin + pi < A.n_pw);
                        const int w = s_pw[Q.part_begin + pi];
                        jp = w >= 0 ? S + w : cinst + ~w;
                        mov = w >= 0;
                    } else {
                        const int jj = P.partners[Q.part_begin + pi];
                        jp = inst(jj);
                        mov = P.inst[jj].xoff >= 0;
                    }
                    jcp += pairs_vs_instance<G, NSO>(qe, jp + 16, *reinterpret_cast<const float4*>(jp + 12), lam_cp, gq,
                        [&](Wrench& pw) { flush_partner<G, GS>(pw, mov, jp + 48, gl); }, smooth);
                }
                finish_term<M>(P, A, sink, Q.term_cp, term_sum<M, GS>(jcp), gl, active, p, s_counts);
            }
            if (G) {
#pragma unroll
                for (int u = 0; u < NSO; ++u)
                    if (gl + GS * u < no) own.add_point(wq[u][0], wq[u][1], wq[u][2], gq[u][0], gq[u][1], gq[u][2]);
                own.template group_sum<GS>();
                if (gl == 0) add_wrench(oip + 48, own);
            }
        }

        // ---- phase D: soft costs (Eq. 2 second sum) ----
        if (P.n_goal > 1) {   // MinimizeObjDist: sum_{i<j} ||P_i - P_j||  (Listing 2 obj_dist)
            for (int a = 0; a < P.n_goal; ++a) {
                for (int b = a + 1; b < P.n_goal; ++b) {
                    const float* pa = ipose(P.goal_inst[a]);
                    const float* pb = ipose(P.goal_inst[b]);
                    const float dx = pa[3] - pb[3], dy = pa[7] - pb[7], dz = pa[11] - pb[11];
                    const float d = sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
                    soft = fmaf(P.lam_goal, d, soft);
                    if (G && gl == 0 && d > 0.f) {
                        const float k = P.lam_goal / d;
                        const int ia = P.goal_inst[a], ib = P.goal_inst[b];
                        if (P.inst[ia].xoff >= 0) {
                            float* t = iwr(ia);
                            t[0] += dx * k; t[1] += dy * k; t[2] += dz * k;
                            t[3] += pa[7] * dz * k - pa[11] * dy * k;
                            t[4] += pa[11] * dx * k - pa[3] * dz * k;
                            t[5] += pa[3] * dy * k - pa[7] * dx * k;
                        }
                        if (P.inst[ib].xoff >= 0) {
                            float* t = iwr(ib);
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
            // (each knot's coordinates read once: the segment's end becomes the next segment's start)
            float prev[NJL];
#pragma unroll
            for (int u = 0; u < NJL; ++u) prev[u] = val(0, gl + GS * u);
            for (int j = 0; j < nseg; ++j) {
                float dlt[NJL], s2 = 0.f;
#pragma unroll
                for (int u = 0; u < NJL; ++u) {
                    const int jt = gl + GS * u;
                    const float cur = val(j + 1, jt);
                    dlt[u] = cur - prev[u];
                    prev[u] = cur;
                    s2 = fmaf(dlt[u], dlt[u], s2);
                }
                const float len = sqrtf(gsum<GS>(s2));
                soft = fmaf(P.lam_traj, len, soft);
                if (G && len > 0.f) {
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
        if (G) {
            __syncwarp();
            for (int i = 0; i < P.n_inst; ++i) {
                const KInst& I = P.inst[i];
                if (I.xoff < 0) continue;
                const float* wr = iwr(i);
                if (gl < 3) {
                    gs[I.xoff + gl] += wr[gl];
                } else if (gl == 3) {   // d/dyaw = z . (M - t x F)
                    const float tx = xs[I.xoff], ty = xs[I.xoff + 1];
                    gs[I.xoff + 3] += wr[5] - (tx * wr[1] - ty * wr[0]);
                }
            }
            __syncwarp();
        }

        if (M == MODE_EVAL) {
            if (active) {
                if (gl == 0 && A.out_J) A.out_J[p] = Jtot;
                if (gl == 0 && A.out_soft) A.out_soft[p] = soft;
                if (A.out_grad) for (int d = gl; d < D; d += GS) A.out_grad[p * D + d] = gs[d];
            }
        } else if (M == MODE_CHECK) {
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
            const float rbc1 = A.rbc1[it];
            const float rbc2 = A.rbc2[it];
            if (!invalid) {
                for (int d = gl; d < D; d += GS) {
                    const float g = gs[d] * P.grad_scale;
                    const float mm = fmaf(P.beta1, A.m[p * D + d], (1.f - P.beta1) * g);
                    const float vv = fmaf(P.beta2, A.v[p * D + d], (1.f - P.beta2) * g * g);
                    if (active) { A.m[p * D + d] = mm; A.v[p * D + d] = vv; }
                    const float mh = mm * rbc1;
                    const float vh = vv * rbc2;
                    const float xn = xs[d] - A.lr[d] * mh / (sqrtf(vh) + P.adam_eps);
                    xs[d] = fminf(fmaxf(xn, A.lo[d]), A.hi[d]);
                }
            }
            __syncwarp();
        }
    };
    for (int it = 0; it < n_iter; ++it) iteration(std::integral_constant<int, MODE>{}, it);
    if constexpr (MODE == MODE_OPT) {
        // Eq. 3 check of the state after the last step, in the same launch (tamp_optimize_and_check): no second
        // launch re-loading the state and re-building the instances
        if (A.check_after) {
            if (BSYNC > 0) __syncthreads();
            iteration(std::integral_constant<int, MODE_CHECK>{}, n_iter);
        }
    }

    if (MODE == MODE_OPT && active) {
        for (int d = gl; d < D; d += GS) A.x[p * D + d] = xs[d];
        if (gl == 0) A.invalid[p] = invalid ? 1 : 0;
    }
    if (MODE == MODE_CHECK || (MODE == MODE_OPT && A.check_after)) {
        __syncthreads();
        for (int i = threadIdx.x; i < P.n_terms + 2; i += blockDim.x)
            if (s_counts[i]) atomicAdd(&A.out_counts[i], s_counts[i]);
    }
}

}  // namespace tamp
