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

#include <algorithm>
#include <atomic>

#include "particle.cuh"

namespace tamp {
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

__device__ __forceinline__ void uniform4(uint64_t seed, uint64_t gidx, uint32_t var, int block, float u[4]) {
    const uint4 w = philox4x32_10(make_uint4((uint32_t)gidx, (uint32_t)(gidx >> 32), var, (uint32_t)block),
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
        if (V.kind == KS_GRASP) {       // grasps in the object frame, frozen
            uniform4(seed, gidx, V.stream, 0, u);
            const float gxy = V.a[0];
            float* g = grasp + (i * SP.n_grasp + V.slot) * 12;
            const bool six = V.a[2] > 0.5f;
            const int face = six ? min((int)floorf(u[0] * 5.f), 4) : 0;
            const float* uu = six ? u + 1 : u;          // 6-DOF: u0 picks the face
            const float gx = -gxy + 2.f * gxy * uu[0];
            const float gy = -V.a[3] + 2.f * V.a[3] * uu[1];
            const float gamma = -kPi + 2.f * kPi * uu[2];
            float s, c;
            sincosf(gamma, &s, &c);
            if (face == 0) {   // top-down: Trans(gx, gy, gz) Rz(gamma) Rx(pi)
                g[0] = c;   g[1] = s;   g[2] = 0.f;  g[3] = gx;
                g[4] = s;   g[5] = -c;  g[6] = 0.f;  g[7] = gy;
                g[8] = 0.f; g[9] = 0.f; g[10] = -1.f; g[11] = V.a[1];
            } else {           // side: Trans(0, 0, gz) R_face Rz(gamma), approach axis = -n_face
                float R[9];
                if (face == 1) { const float r[9] = {0.f, 0.f, -1.f, s, c, 0.f, c, -s, 0.f}; for (int k = 0; k < 9; ++k) R[k] = r[k]; }
                else if (face == 2) { const float r[9] = {0.f, 0.f, 1.f, s, c, 0.f, -c, s, 0.f}; for (int k = 0; k < 9; ++k) R[k] = r[k]; }
                else if (face == 3) { const float r[9] = {c, -s, 0.f, 0.f, 0.f, -1.f, s, c, 0.f}; for (int k = 0; k < 9; ++k) R[k] = r[k]; }
                else { const float r[9] = {c, -s, 0.f, 0.f, 0.f, 1.f, -s, -c, 0.f}; for (int k = 0; k < 9; ++k) R[k] = r[k]; }
                g[0] = R[0]; g[1] = R[1]; g[2] = R[2];  g[3] = 0.f;
                g[4] = R[3]; g[5] = R[4]; g[6] = R[5];  g[7] = 0.f;
                g[8] = R[6]; g[9] = R[7]; g[10] = R[8]; g[11] = V.a[1];
            }
        } else if (V.kind == KS_PLACEMENT) {   // uniform on the surface region shrunk by the footprint
            uniform4(seed, gidx, V.stream, 0, u);
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
            uniform4(seed, gidx, V.stream, 0, u);
            uniform4(seed, gidx, V.stream, 1, u + 4);
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
// T(p) T(g), one thread per (particle, conf) pair, then the knots are re-interpolated from the refined endpoint
// confs.
//   e = [t* - t_ee ; rotvec(R* R_ee^T)],  J = [z_j x (t_ee - o_j) ; z_j],  dq = J^T (J J^T + mu^2 I)^-1 e
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ void chol6_solve(float A[21], const float b[6], float y[6]) {
    // A: packed lower triangle, row-major (i, j <= i) -> index i*(i+1)/2 + j.  In-place Cholesky.  (Every loop has
    // a constant trip count with a guard: nvcc left an inner loop with a j-dependent bound rolled, which put A in
    // local memory.)
#pragma unroll
    for (int j = 0; j < 6; ++j) {
        float d = A[j * (j + 1) / 2 + j];
#pragma unroll
        for (int k = 0; k < 6; ++k)
            if (k < j) d = fmaf(-A[j * (j + 1) / 2 + k], A[j * (j + 1) / 2 + k], d);
        const float ljj = sqrtf(fmaxf(d, 1e-30f));
        const float inv = 1.f / ljj;
        A[j * (j + 1) / 2 + j] = ljj;
#pragma unroll
        for (int i = 0; i < 6; ++i) {
            if (i <= j) continue;
            float v = A[i * (i + 1) / 2 + j];
#pragma unroll
            for (int k = 0; k < 6; ++k)
                if (k < j) v = fmaf(-A[i * (i + 1) / 2 + k], A[j * (j + 1) / 2 + k], v);
            A[i * (i + 1) / 2 + j] = v * inv;
        }
    }
    float z[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) {     // L z = b
        float v = b[i];
#pragma unroll
        for (int k = 0; k < 6; ++k)
            if (k < i) v = fmaf(-A[i * (i + 1) / 2 + k], z[k], v);
        z[i] = v / A[i * (i + 1) / 2 + i];
    }
#pragma unroll
    for (int i = 5; i >= 0; --i) {    // L^T y = z
        float v = z[i];
#pragma unroll
        for (int k = 0; k < 6; ++k)
            if (k > i) v = fmaf(-A[k * (k + 1) / 2 + i], y[k], v);
        y[i] = v / A[i * (i + 1) / 2 + i];
    }
}

// One thread per (particle, conf, seed): the Kin-constrained confs are independent given the sampled grasps and
// placements (grid.y = conf), and the S restarts of a conf (R6) run on S adjacent lanes.  The chain is
// composed once per iteration; the joint axes z_j and origins o_j of the forward pass stay in registers for
// J J^T = sum_j c_j c_j^T, c_j = [z_j x (t_ee - o_j) ; z_j], and for dq_j = c_j . y.  (An earlier 8-lanes-per-pair
// mapping with the FK product scan repeated the 6x6 solve on every lane of the group: 4.4x slower at config 2,
// profiles/README.md.)
struct KIkStreams { uint32_t stream[TAMP_MAX_FK]; };   // Philox stream of each Kin conf's sampler
constexpr float kIkTolPos = 1e-3f, kIkTolRot = 1e-3f;  // a restart counts as converged below both
constexpr int kIkRestartsPerRound = 2;                   // restarts per pair and round of k_ik_restarts

// tool pose of the chain at q, and the Kin errors to T*: e_pos = ||t* - t_ee||, theta = angle(R* R_ee^T)
// (joint 1 from its fixed transform, which carries the base; joints 2..7 as modified-DH steps on the packed frame,
// dh_fwd; the joint axes z_j and origins o_j are frame j's third column and translation)
__device__ __forceinline__ void ik_fk(const KProgram& P, const float (&q)[TAMP_NJ], M34& T, float (&z)[TAMP_NJ][3],
                                      float (&o)[TAMP_NJ][3]) {
    M34P Tp;
#pragma unroll
    for (int j = 0; j < TAMP_NJ; ++j) {
        float s, c;
        fsincos(q[j], &s, &c);
        if (j == 0) {
            M34 A0;
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                const float* Fr = P.F[0] + 4 * i;
                A0.r[3 * i] = fmaf(Fr[0], c, Fr[1] * s);
                A0.r[3 * i + 1] = fmaf(Fr[1], c, -Fr[0] * s);
                A0.r[3 * i + 2] = Fr[2];
                A0.t[i] = Fr[3];
            }
            Tp = pack_m34(A0);
        } else {
            dh_fwd(Tp, P.dh[j], c, s);
        }
        z[j][0] = lo(Tp.r01[2]); z[j][1] = hi(Tp.r01[2]); z[j][2] = Tp.r2[2];
        o[j][0] = lo(Tp.t01); o[j][1] = hi(Tp.t01); o[j][2] = Tp.t2;
    }
    M34 Fe;
    load_m34(Fe, P.F[kGroup - 1]);
    T = unpack_m34(compose_p(Tp, Fe));
}

__device__ __forceinline__ void ik_error(const M34& Ts, const M34& T, float (&e)[6], float& epos, float& th) {
    e[0] = Ts.t[0] - T.t[0]; e[1] = Ts.t[1] - T.t[1]; e[2] = Ts.t[2] - T.t[2];
    float E[9];   // R* R_ee^T
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            E[3 * i + j] = fmaf(Ts.r[3 * i], T.r[3 * j], fmaf(Ts.r[3 * i + 1], T.r[3 * j + 1], Ts.r[3 * i + 2] * T.r[3 * j + 2]));
    const float wx = E[7] - E[5], wy = E[2] - E[6], wz = E[3] - E[1];
    const float wn = sqrtf(fmaf(wx, wx, fmaf(wy, wy, wz * wz)));
    th = fatan2_pos(0.5f * wn, 0.5f * (E[0] + E[4] + E[8] - 1.f));
    const float kk = wn > 0.f ? th / wn : 0.f;
    e[3] = wx * kk; e[4] = wy * kk; e[5] = wz * kk;
    epos = sqrtf(fmaf(e[0], e[0], fmaf(e[1], e[1], e[2] * e[2])));
}

// DLS iterations from q (in place)
__device__ __forceinline__ void ik_iterate(const KProgram& P, const M34& Ts, float (&q)[TAMP_NJ], int iters, float damp2) {
    float z[TAMP_NJ][3], o[TAMP_NJ][3], e[6], epos, th;
    M34 T;
    for (int it = 0; it < iters; ++it) {
        ik_fk(P, q, T, z, o);
        ik_error(Ts, T, e, epos, th);
        auto column = [&](int j, float (&c)[6]) {
            const float rx = T.t[0] - o[j][0], ry = T.t[1] - o[j][1], rz = T.t[2] - o[j][2];
            c[0] = z[j][1] * rz - z[j][2] * ry; c[1] = z[j][2] * rx - z[j][0] * rz; c[2] = z[j][0] * ry - z[j][1] * rx;
            c[3] = z[j][0]; c[4] = z[j][1]; c[5] = z[j][2];
        };
        float A[21];
#pragma unroll
        for (int i = 0; i < 21; ++i) A[i] = 0.f;
#pragma unroll
        for (int j = 0; j < TAMP_NJ; ++j) {
            float c[6];
            column(j, c);
#pragma unroll
            for (int a = 0; a < 6; ++a)
#pragma unroll
                for (int b = 0; b <= a; ++b) A[a * (a + 1) / 2 + b] = fmaf(c[a], c[b], A[a * (a + 1) / 2 + b]);
        }
#pragma unroll
        for (int a = 0; a < 6; ++a) A[a * (a + 1) / 2 + a] += damp2;
        float y[6];
        chol6_solve(A, e, y);
#pragma unroll
        for (int j = 0; j < TAMP_NJ; ++j) {
            float c[6];
            column(j, c);
            const float dq = fmaf(c[0], y[0], fmaf(c[1], y[1], fmaf(c[2], y[2], fmaf(c[3], y[3], fmaf(c[4], y[4], c[5] * y[5])))));
            q[j] = fminf(fmaxf(q[j] + dq, P.jlo[j]), P.jhi[j]);
        }
    }
}

// final errors of q: converged (<= kIkTolPos, kIkTolRot) and the restart score e_pos + theta
__device__ __forceinline__ bool ik_final(const KProgram& P, const M34& Ts, const float (&q)[TAMP_NJ], float& score) {
    float z[TAMP_NJ][3], o[TAMP_NJ][3], e[6], epos, th;
    M34 T;
    ik_fk(P, q, T, z, o);
    ik_error(Ts, T, e, epos, th);
    score = epos + th;
    return epos <= kIkTolPos && th <= kIkTolRot;
}

// the Kin conf of grid row blockIdx.y: its KFk and the target T* = T(p) T(g) of particle p
__device__ __forceinline__ bool ik_target(const KProgram& P, const float* xp, const float* grasp, int64_t p, KFk& K, M34& Ts) {
    int fsel = -1, nth = 0;
    for (int f = 0; f < P.n_fk && fsel < 0; ++f) {
        if ((P.fk[f].term_kp < 0 && P.fk[f].term_kr < 0) || P.fk[f].ghost) continue;
        if (nth++ == (int)blockIdx.y) fsel = f;
    }
    if (fsel < 0) return false;
    K = P.fk[fsel];
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
    Ts = compose(Tp, Tg);
    return true;
}

// Stage A: restart 0 of every (particle, conf) pair from its uniform sample.  With restarts (list != nullptr),
// pairs that did not converge are appended to the conf's list (warp-aggregated atomics; the order of a list
// does not affect any result).
__global__ void __launch_bounds__(128) k_ik(const __grid_constant__ KProgram P, float* __restrict__ x,
                                            const float* __restrict__ grasp, int64_t n, int iters, float damp2,
                                            int32_t* __restrict__ list, int32_t* __restrict__ list_n,
                                            float* __restrict__ best) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    float* xp = x + p * P.D;
    KFk K;
    M34 Ts;
    if (!ik_target(P, xp, grasp, p, K, Ts)) return;
    float q[TAMP_NJ];
#pragma unroll
    for (int j = 0; j < TAMP_NJ; ++j) q[j] = xp[K.xoff + j];
    ik_iterate(P, Ts, q, iters, damp2);
#pragma unroll
    for (int j = 0; j < TAMP_NJ; ++j) xp[K.xoff + j] = q[j];
    if (list) {
        float score;
        const bool fail = !ik_final(P, Ts, q, score);
        const unsigned m = __ballot_sync(__activemask(), fail);
        if (fail) {
            const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
            int base = 0;
            if (lane == leader) base = atomicAdd(&list_n[blockIdx.y], __popc(m));
            base = __shfl_sync(m, base, leader);
            list[(int64_t)blockIdx.y * n + base + __popc(m & ((1u << lane) - 1u))] = (int32_t)p;
            best[(int64_t)blockIdx.y * n + p] = score;      // restart 0's score: the best so far
        }
    }
}

// Stage B, one round: restarts s0 .. s0+R-1 of the pairs still unconverged (list_in), on R adjacent lanes.  A
// pair whose round has a converged restart keeps the first one and is done; otherwise the round's best restart
// replaces the kept conf only if its score is strictly lower than the best so far (earlier restarts win ties,
// a number beats NaN), and the pair goes on to the next round's list.  Rounds run in restart order, so the
// result equals running all restarts of every pair and keeping the first converged, else the lowest score
// (lowest index on ties), while most pairs stop after their first rounds.
template <int R>
__global__ void __launch_bounds__(128) k_ik_restarts(const __grid_constant__ KProgram P, const KIkStreams Z,
                                                     float* __restrict__ x, const float* __restrict__ grasp, int64_t n,
                                                     int64_t gofs, uint64_t seed, int iters, float damp2, int s0,
                                                     int s_end, const int32_t* __restrict__ list_in, const int32_t* __restrict__ n_in,
                                                     int32_t* __restrict__ list_out, int32_t* __restrict__ n_out,
                                                     float* __restrict__ best) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int sl = (int)(threadIdx.x & (R - 1));
    const int sd = s0 + sl;                                         // restart index
    const int64_t cnt = n_in[blockIdx.y];
    if ((int64_t)blockIdx.x * blockDim.x / R >= cnt) return;       // block-uniform: past the list
    const bool active = t / R < cnt;
    const int64_t e = active ? t / R : cnt - 1;                    // idle lanes mirror the last entry (shuffles)
    const int64_t p = list_in[(int64_t)blockIdx.y * n + e];
    float* xp = x + p * P.D;
    KFk K;
    M34 Ts;
    if (!ik_target(P, xp, grasp, p, K, Ts)) return;
    const bool valid = sd < s_end;                                  // lanes past the last restart pad the round
    float q[TAMP_NJ];
    {
        float u[8];
        uniform4(seed, (uint64_t)(gofs + p), Z.stream[blockIdx.y], 2 * sd, u);
        uniform4(seed, (uint64_t)(gofs + p), Z.stream[blockIdx.y], 2 * sd + 1, u + 4);
#pragma unroll
        for (int j = 0; j < TAMP_NJ; ++j) q[j] = P.jlo[j] + u[j] * (P.jhi[j] - P.jlo[j]);
    }
    float score = INFINITY;
    bool conv = false;
    if (valid) {
        ik_iterate(P, Ts, q, iters, damp2);
        conv = ik_final(P, Ts, q, score);
    }
    const unsigned lane0 = threadIdx.x & 31 & ~(unsigned)(R - 1);
    const unsigned cm = (__ballot_sync(FULL, conv) >> lane0) & ((1u << R) - 1u);
    if (cm) {                                                       // first converged restart of the round
        if (active && sl == __ffs(cm) - 1) {
#pragma unroll
            for (int j = 0; j < TAMP_NJ; ++j) xp[K.xoff + j] = q[j];
        }
        return;
    }
    // the round's best restart: smallest score (NaN and padding lanes count as +inf), lowest index on ties --
    // a total order, so exactly one lane of the pair wins
    float bs = score == score ? score : INFINITY;
    int bi = sl;
#pragma unroll
    for (int m = 1; m < R; m <<= 1) {
        const float ob = __shfl_xor_sync(FULL, bs, m, R);
        const int oi = __shfl_xor_sync(FULL, bi, m, R);
        if (ob < bs || (ob == bs && oi < bi)) { bs = ob; bi = oi; }
    }
    if (!active || sl != bi) return;
    float* bp = best + (int64_t)blockIdx.y * n + p;
    const float prev = *bp == *bp ? *bp : INFINITY;
    if (bs < prev) {
        *bp = bs;
#pragma unroll
        for (int j = 0; j < TAMP_NJ; ++j) xp[K.xoff + j] = q[j];
    }
    if (list_out) {                                                 // still unconverged: next round
        const int o = atomicAdd(&n_out[blockIdx.y], 1);
        list_out[(int64_t)blockIdx.y * n + o] = (int32_t)p;
    }
}

// knots: linear interpolation between the (IK-refined) endpoint confs; 8 lanes per particle
__global__ void __launch_bounds__(128) k_knots(const __grid_constant__ KProgram P, float* __restrict__ x, int64_t n) {
    const int gl = threadIdx.x & (kGroup - 1);
    const int64_t p = (int64_t)blockIdx.x * (blockDim.x / kGroup) + threadIdx.x / kGroup;
    if (p >= n || gl >= TAMP_NJ) return;
    float* xp = x + p * P.D;
    for (int tr = 0; tr < P.n_traj; ++tr) {
        const KTraj& Tj = P.traj[tr];
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
constexpr int kSortChunkSmall = 256;

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
template <int C>   // chunk size (power of two); C / 2 threads, one compare-exchange each per stage
__global__ void __launch_bounds__(C / 2) k_sort_chunk(const unsigned long long* __restrict__ kin, const int32_t* __restrict__ pin,
                                                     int64_t n, int k, unsigned long long* __restrict__ kout,
                                                     int32_t* __restrict__ pout) {
    __shared__ unsigned long long sk[C];
    __shared__ int32_t sp[C];
    const int64_t base = (int64_t)blockIdx.x * C;
    for (int i = threadIdx.x; i < C; i += blockDim.x) {
        const int64_t g = base + i;
        sk[i] = g < n ? kin[g] : ~0ull;
        sp[i] = g < n ? pin[g] : -1;
    }
    __syncthreads();
    for (int size = 2; size <= C; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const int i = threadIdx.x;
            const int lo = 2 * i - (i & (stride - 1));
            const int hi = lo + stride;
            const bool up = ((lo & size) == 0);
            const unsigned long long a = sk[lo], b = sk[hi];
            if ((a > b) == up) {
                sk[lo] = b; sk[hi] = a;
                const int32_t t = sp[lo]; sp[lo] = sp[hi]; sp[hi] = t;
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
void note_launch();

// Adam moments [n][D] <-> the serial mapping's 32-particle tiles (tamp_get_state / tamp_set_state)
__global__ void k_mv_layout(const float* __restrict__ src, float* __restrict__ dst, int64_t n, int D, int to_w32) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * D) return;
    const int64_t p = e / D;
    const int d = (int)(e - p * D);
    const int64_t w = mv_w32_index(p, d, D);
    if (to_w32) dst[w] = src[e];
    else dst[e] = src[w];
}

cudaError_t launch_mv_layout(const float* src, float* dst, int64_t n, int D, int to_w32, cudaStream_t st) {
    if (n <= 0 || D <= 0) return cudaSuccess;
    k_mv_layout<<<(unsigned)((n * D + 255) / 256), 256, 0, st>>>(src, dst, n, D, to_w32);
    note_launch();
    return cudaGetLastError();
}

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
static inline void counted() { note_launch(); }

cudaError_t launch_particle_sm(bool smooth, int mode, int gs, int bsync, int threads, const KProgram& P, const KArgs& A,
                               size_t smem, cudaStream_t st);
int particle_kernel_regs_sm(int gs, int threads);

// gs = lanes per particle: 1 (serial mapping), 4 (two link frames per lane), 8 (one), 16 (two FK instances);
// threads = block size (multiple of 32, <= 768); smem sized for threads / gs particles;
// bsync = block-synchronisation level (see k_particle).
cudaError_t launch_particle_serial(bool smooth, int mode, int threads, const KProgram& P, const KArgs& A,
                                   cudaStream_t st);

cudaError_t launch_particle(int mode, int gs, int bsync, int threads, const KProgram& P, const KArgs& A, size_t smem,
                            cudaStream_t st) {
    if (A.n <= 0) return cudaSuccess;
    if (gs == 1) return launch_particle_serial(P.smooth > 0.f, mode, threads, P, A, st);
    return launch_particle_sm(P.smooth > 0.f, mode, gs, bsync, threads, P, A, smem, st);
}

// registers per thread of the hot kernel (for the launch-configuration policy)
int particle_kernel_regs(int gs, int threads) { return particle_kernel_regs_sm(gs, threads); }

cudaError_t launch_ik(const KProgram& P, const KSampleProgram& SP, float* x, const float* grasp, int64_t n, int64_t gofs,
                      uint64_t seed, int iters, float damping, int n_seeds, int32_t* lists, int32_t* list_n,
                      float* best, cudaStream_t st) {
    if (n <= 0 || iters <= 0) return cudaSuccess;
    KIkStreams Z;
    int n_kin = 0;
    for (int f = 0; f < P.n_fk; ++f) {
        if ((P.fk[f].term_kp < 0 && P.fk[f].term_kr < 0) || P.fk[f].ghost) continue;
        Z.stream[n_kin] = 0u;
        for (int v = 0; v < SP.n_vars; ++v)      // the conf sampler that drew this conf (restart 0's start)
            if (SP.v[v].kind == KS_CONF && SP.v[v].xoff == P.fk[f].xoff) Z.stream[n_kin] = SP.v[v].stream;
        ++n_kin;
    }
    const int per_block = 128 / kGroup;
    const unsigned bx = (unsigned)((n + per_block - 1) / per_block);
    if (n_kin > 0) {
        const float d2 = damping * damping;
        const bool restarts = n_seeds > 1;
        // lists[2][n_kin][n] (ping-pong), list_n[rounds + 1][n_kin]; rounds of 2 restarts (rounds of 4 measured
        // no faster at config 2 and slower for 64K-1M pairs: most pairs converge within their first restarts)
        const int per_round = kIkRestartsPerRound;
        const int rounds = restarts ? (n_seeds - 1 + per_round - 1) / per_round : 0;
        if (restarts) {
            const cudaError_t e = cudaMemsetAsync(list_n, 0, sizeof(int32_t) * n_kin * (rounds + 1), st);
            if (e != cudaSuccess) return e;
        }
        k_ik<<<dim3((unsigned)((n + 127) / 128), (unsigned)n_kin), 128, 0, st>>>(P, x, grasp, n, iters, d2,
                                                                                restarts ? lists : nullptr, list_n, best);
        counted();
        for (int r = 0; r < rounds; ++r) {
            const int s0 = 1 + r * per_round;
            const int R = n_seeds - s0 >= 2 ? 2 : 1;
            int32_t* lin = lists + (size_t)(r & 1) * n_kin * n;
            int32_t* lout = r + 1 < rounds ? lists + (size_t)((r + 1) & 1) * n_kin * n : nullptr;
            // grid sized for the worst case (every pair unconverged); blocks past the list exit at once
            const dim3 grid((unsigned)((n * R + 127) / 128), (unsigned)n_kin);
            int32_t* nin = list_n + r * n_kin;
            int32_t* nout = list_n + (r + 1) * n_kin;
            if (R >= 2)
                k_ik_restarts<2><<<grid, 128, 0, st>>>(P, Z, x, grasp, n, gofs, seed, iters, d2, s0, n_seeds, lin, nin, lout, nout, best);
            else
                k_ik_restarts<1><<<grid, 128, 0, st>>>(P, Z, x, grasp, n, gofs, seed, iters, d2, s0, n_seeds, lin, nin, lout, nout, best);
            counted();
        }
    }
    if (P.n_traj > 0) {
        k_knots<<<bx, 128, 0, st>>>(P, x, n);
        counted();
    }
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
    // small k: 256-key chunks (36 short block-barrier stages, many blocks per pass); else 2048-key chunks
    const bool small = k <= kSortChunkSmall / 4;
    const int64_t C = small ? kSortChunkSmall : kSortChunk;
    do {
        const int64_t chunks = (cnt + C - 1) / C;
        const int keep = (int)(cnt < k ? cnt : k);
        if (small)
            k_sort_chunk<kSortChunkSmall><<<(unsigned)chunks, kSortChunkSmall / 2, 0, st>>>(ki, pi, cnt, keep, ko, po);
        else
            k_sort_chunk<kSortChunk><<<(unsigned)chunks, kSortChunk / 2, 0, st>>>(ki, pi, cnt, keep, ko, po);
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
