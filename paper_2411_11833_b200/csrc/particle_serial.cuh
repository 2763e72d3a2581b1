// particle_serial.cuh -- the serial mapping of K2 / K3 / eval: one thread per particle.
//
// The lane mapping (particle.cuh) spreads a particle over 4-16 lanes, which hides latency when particles
// are few but repeats the per-particle serial work (FK scan steps, Kin, bookkeeping) on every lane of the
// group.  When a launch holds many waves of particles of a small skeleton (config 1 at 2^17-2^20
// particles), one thread per particle does the minimal work: the chain is composed once, no shuffles.
//
// Per FK instance, without storing the link frames: forward T_1 .. T_8 (= tool), Kin at T_8, then a
// backward sweep over the links 8 -> 1 recovering T_{l-1} = T_l Rz(-q_l) F_l^{-1} while it evaluates
// that link's spheres and accumulates the suffix wrench (F, M) of all links >= l, so that
// dJ/dq_l = z_l . (M - o_l x F) is available exactly when joint l is reached.
// Per-thread state (x, Adam moments, gradient, grasps, instance poses and wrenches) lives in shared memory, one
// row per thread (field f of thread t at [t * pitch + f], pitch odd: a warp reading one field is conflict-free).
// Supported: every term except SELF and held objects at knots (tamp_api.cu selects the lane mapping then).
#pragma once
#include "particle.cuh"

namespace tamp {

struct SerialLayout {
    int x, g, gT, ipose, iwr, n;   // column offsets (floats per thread)
};

// The Adam moments are not in the rows: they stay in global memory (L2-resident for the launch) in the 32-particle
// tile layout of the serial mapping (mv_w32_index), read and written once per step by Adam -- which frees 2 D floats
// of shared memory per particle for more resident warps.
__host__ __device__ inline SerialLayout serial_layout(const KProgram& P, bool /*mv*/ = true) {
    SerialLayout L;
    int f = 0;
    L.x = f;     f += P.D;
    L.g = f;     f += P.D;
    L.gT = f;    f += 12 * P.n_grasp;
    L.ipose = f; f += 8 * P.n_inst;    // cos, sin, px, py, pz, world bounding-sphere centre xyz
    int nm = 0;                        // movable instances (slot = index among them)
    for (int i = 0; i < P.n_inst; ++i) nm += P.inst[i].xoff >= 0;
    L.iwr = f;   f += 6 * nm;          // wrench (F, M about the world origin) on each movable instance
    L.n = f;
    return L;
}

constexpr int kSerialThreads = 512;   // launch bound (blocks of <= 512 threads, <= 128 registers)
#ifndef TAMP_SERIAL_MAXT_PP
#define TAMP_SERIAL_MAXT_PP 640          // pick-place variant: <= 102 registers
#endif
constexpr int kSerialThreadsPP = TAMP_SERIAL_MAXT_PP;

// floats per thread row of the shared-memory state: the layout's size rounded up to odd, so that the 32 threads
// of a warp reading the same field (stride = row pitch) hit 32 distinct banks
__host__ __device__ inline int serial_row_pitch(const SerialLayout& L) { return L.n | 1; }

// dynamic shared memory of a serial-mapping block of `threads` particles (one row per thread)
// (+ the Adam step sizes and bounds lr, lo, hi of the D coordinates once per block in optimisation mode)
__host__ __device__ inline size_t serial_smem_bytes(const KProgram& P, int threads, bool mv) {
    return ((size_t)serial_row_pitch(serial_layout(P, mv)) * threads + (mv ? 3 * P.D : 0)) * sizeof(float);
}

// term bookkeeping: warp-aggregated counts (every thread of the warp calls it for the same term)
template <int MODE>
__device__ __forceinline__ void serial_term(const KProgram& P, const KArgs& A, TermSink<MODE>& sink, int term, float val,
                                            bool active, int64_t p, int* s_counts) {
    sink.J = fmaf(P.term_lam[term], val, sink.J);
    if (MODE == MODE_EVAL) {
        if (active && A.out_Jc) A.out_Jc[p * P.n_terms + term] = val;
    } else if (MODE == MODE_CHECK) {
        const bool ok = val <= P.term_eps[term];
        sink.sat = sink.sat && ok;
        const unsigned b = __ballot_sync(FULL, active && ok);
        if ((threadIdx.x & 31) == 0 && b) atomicAdd(&s_counts[term], __popc(b));
    }
}

// Is the program of the pick-place class (PP): every configuration's robot collision is against at most one
// axis-aligned box and no partner instances (config 1)?  Then k_serial<.., PP = true> unrolls the link sweep (the per-link robot data
// become constant-bank operands: no indexed constant loads or loop control) and keeps only the packed one-box path.
__host__ __device__ inline bool serial_program_pp(const KProgram& P) {
    for (int f = 0; f < P.n_fk; ++f) {
        const KFk& K = P.fk[f];
        if (K.ghost || K.term_cf < 0) continue;
        if (K.part_count != 0 || (K.obb_mask & (K.obb_mask - 1)) != 0) return false;
        for (int b = 0; b < TAMP_MAX_OBB; ++b)
            if (((K.obb_mask >> b) & 1) && !P.obb[b].aligned) return false;
    }
    return true;
}

#ifndef TAMP_SERIAL_CONF_BARRIER   // block barrier after every configuration (1) or only after the Place terms (0);
#define TAMP_SERIAL_CONF_BARRIER 0 // the generic sweep keeps it (its larger body: the instruction cache)
#endif

#ifndef TAMP_SERIAL_ADAM_BATCH      // coordinates whose moments are loaded together (one L2 latency per batch)
#define TAMP_SERIAL_ADAM_BATCH 6
#endif

#ifndef TAMP_SERIAL_LINK_BROAD     // PP sweep: gate each link's packed sphere tests by its bounding sphere
#define TAMP_SERIAL_LINK_BROAD 1
#endif

template <int MODE, bool SMOOTH, bool PP>
__global__ void __launch_bounds__(PP ? kSerialThreadsPP : kSerialThreads, 1) k_serial(const __grid_constant__ KProgram P, const KArgs A) {
    constexpr bool GRAD = MODE != MODE_CHECK;
    const float smooth = SMOOTH ? P.smooth : 0.f;
    extern __shared__ float4 smem4[];
    __shared__ float4 s_osph[TAMP_MAX_OBJECTS][TAMP_MAX_OBJ_SPHERES];
    __shared__ int s_counts[TAMP_MAX_TERMS + 2];
    float* S = reinterpret_cast<float*>(smem4);
    const int NT = blockDim.x, tid = threadIdx.x;
    const int64_t pid = (int64_t)blockIdx.x * NT + tid;
    const bool active = pid < A.n;
    const int64_t p = active ? pid : (A.n - 1);
    const SerialLayout L = serial_layout(P, MODE == MODE_OPT);
    const int D = P.D;
    // per-thread state rows (odd pitch: a warp reading one field of its 32 rows is conflict-free); every field
    // access is my row base + a warp-uniform offset
    const int ROWP = serial_row_pitch(L);
    TAMP_DCHECK((tid + 1) * ROWP <= A.smem_floats);
    float* const Sr = S + tid * ROWP;
    auto col = [&](int f) -> float& { return Sr[f]; };
    // block-cooperative, coalesced copy between the block's rows of a [n][w] array and fields c0..c0+w of the rows
    const int64_t row0 = (int64_t)blockIdx.x * NT;
    const int nrows = (int)min((int64_t)NT, A.n - row0);
    // element e = row * w + c of the block's rows; (row, c) advanced incrementally (no division per element)
    auto load_rows = [&](const float* src, int w, int c0) {
        const float* base = src + row0 * w;
        const int dq = NT / w, dr = NT % w;
        int q = tid / w, r = tid % w;
        // cp.async (global -> shared, no register round trip): every load of the block is in flight at once
        // instead of one HBM latency per element the thread copies; completed by cp_async_wait_all before the
        // block barrier that ends the prologue
        for (int e = tid; e < nrows * w; e += NT) {
            cp_async4(&S[q * ROWP + c0 + r], base + e);
            q += dq; r += dr;
            if (r >= w) { r -= w; ++q; }
        }
    };
    auto store_rows = [&](float* dst, int w, int c0) {
        float* base = dst + row0 * w;
        const int dq = NT / w, dr = NT % w;
        int q = tid / w, r = tid % w;
        for (int e = tid; e < nrows * w; e += NT) {
            base[e] = S[q * ROWP + c0 + r];
            q += dq; r += dr;
            if (r >= w) { r -= w; ++q; }
        }
    };
    auto xs = [&](int d) -> float& { return col(L.x + d); };
    auto gs = [&](int d) -> float& { return col(L.g + d); };
    auto ip = [&](int i, int k) -> float& { return col(L.ipose + 8 * i + k); };
    auto iw = [&](int i, int k) -> float& { return col(L.iwr + 6 * P.inst[i].slot + k); };   // movable i only
    auto add_iw = [&](int i, const Wrench& w) {
        iw(i, 0) += w.f[0]; iw(i, 1) += w.f[1]; iw(i, 2) += w.f[2];
        iw(i, 3) += w.m[0]; iw(i, 4) += w.m[1]; iw(i, 5) += w.m[2];
    };

    __shared__ float4 s_rsph[kGroup][TAMP_MAX_SPHERES_PER_LINK];
    __shared__ __align__(16) float s_rsoa[kGroup][4 * TAMP_MAX_SPHERES_PER_LINK];   // the same, SoA x[4] y[4] z[4] r[4]
    for (int i = tid; i < TAMP_MAX_OBJECTS * TAMP_MAX_OBJ_SPHERES; i += NT) {
        const int o = i / TAMP_MAX_OBJ_SPHERES, k = i % TAMP_MAX_OBJ_SPHERES;
        s_osph[o][k] = make_float4(P.osph[o][k][0], P.osph[o][k][1], P.osph[o][k][2], P.osph[o][k][3]);
    }
    for (int i = tid; i < kGroup * TAMP_MAX_SPHERES_PER_LINK; i += NT) {
        const int l = i / TAMP_MAX_SPHERES_PER_LINK, k = i % TAMP_MAX_SPHERES_PER_LINK;
        s_rsph[l][k] = make_float4(P.rsph[l][k][0], P.rsph[l][k][1], P.rsph[l][k][2], P.rsph[l][k][3] + P.eta);
#pragma unroll
        for (int c = 0; c < 4; ++c)
            s_rsoa[l][TAMP_MAX_SPHERES_PER_LINK * c + k] = c < 3 ? P.rsph[l][k][c] : P.rsph[l][k][3] + P.eta;
    }
    if (MODE == MODE_CHECK || (MODE == MODE_OPT && A.check_after))
        for (int i = tid; i < P.n_terms + 2; i += NT) s_counts[i] = 0;
    load_rows(A.x, D, L.x);
    if (P.n_grasp) load_rows(A.grasp, 12 * P.n_grasp, L.gT);
    // Adam step sizes and bounds: per-coordinate, the same for every particle (broadcast shared-memory reads)
    float* const s_lr = S + NT * ROWP;
    TAMP_DCHECK(MODE != MODE_OPT || NT * ROWP + 3 * D <= A.smem_floats);
    if (MODE == MODE_OPT)
        for (int i = tid; i < 3 * D; i += NT) s_lr[i] = i < D ? A.lr[i] : (i < 2 * D ? A.lo[i - D] : A.hi[i - 2 * D]);
    bool invalid = A.invalid[p] != 0;
    cp_async_wait_all();
    __syncthreads();

    // world sphere k of an instance at pose (cos, sin, px, py, pz)
    struct IPose { float c, s, x, y, z; };
    auto ipose = [&](int i) -> IPose { return IPose{ip(i, 0), ip(i, 1), ip(i, 2), ip(i, 3), ip(i, 4)}; };
    auto inst_sphere = [&](const IPose& q, int obj, int k) -> float4 {
        const float4 c = s_osph[obj][k];
        return make_float4(fmaf(q.c, c.x, fmaf(-q.s, c.y, q.x)), fmaf(q.s, c.x, fmaf(q.c, c.y, q.y)), q.z + c.z, c.w);
    };
    // one query sphere vs one instance: broad phase on the instance's bounding sphere, then its spheres.
    // Accumulates dJ/dw into g and the partner's reaction into pw (movable partners).
    auto sphere_vs_inst = [&](float wx, float wy, float wz, float rr, int ii, float lam, float* g, Wrench& pw) -> float {
        const int obj = P.inst[ii].obj;
        const float dx = wx - ip(ii, 5), dy = wy - ip(ii, 6), dz = wz - ip(ii, 7);
        const float R = rr + P.obound[obj][3];
        if (fmaf(-R, R, fmaf(dx, dx, fmaf(dy, dy, dz * dz))) >= 0.f) return 0.f;
        float j = 0.f;
        const int no = P.osph_n[obj];
        const IPose q = ipose(ii);
        for (int k = 0; k < no; ++k) {
            const float4 B = inst_sphere(q, obj, k);
            float ux, uy, uz;
            const float pen = sphere_sphere<GRAD>(wx, wy, wz, rr, B, lam, ux, uy, uz, smooth);
            if (pen != 0.f) {
                j += pen;
                if (GRAD) {
                    g[0] -= ux; g[1] -= uy; g[2] -= uz;
                    pw.add_point(B.x, B.y, B.z, ux, uy, uz);
                }
            }
        }
        return j;
    };
    auto sphere_vs_obbs = [&](float wx, float wy, float wz, float rr, uint16_t mask, float lam, float* g) -> float {
        float j = 0.f;
        for (int b = 0; b < P.n_obb; ++b) {
            if (!((mask >> b) & 1)) continue;
            const KObb& B = P.obb[b];
            if (B.rad < kBroadMaxRad) {
                const float dx = wx - B.c[0], dy = wy - B.c[1], dz = wz - B.c[2];
                const float R = rr + B.rad;
                if (fmaf(-R, R, fmaf(dx, dx, fmaf(dy, dy, dz * dz))) >= 0.f) continue;
            }
            j += sphere_obb<GRAD>(wx, wy, wz, rr, B, lam, g[0], g[1], g[2], smooth);
        }
        return j;
    };

    const int n_iter = (MODE == MODE_OPT) ? A.n_steps : 1;
    // one optimisation / check / eval iteration; M = MODE, or MODE_CHECK for the check fused after the last step
    auto iteration = [&](auto mtag, const int it) {
        constexpr int M = decltype(mtag)::value;
        constexpr bool G = M != MODE_CHECK;
        TermSink<M> sink;
        float soft = 0.f;

        // ---- instances: pose, world bounding-sphere centre; zero accumulators ----
        for (int i = 0; i < P.n_inst; ++i) {
            const KInst& I = P.inst[i];
            if (I.xoff >= 0 || it == 0) {
                float px, py, pz, yaw;
                if (I.xoff >= 0) { px = xs(I.xoff); py = xs(I.xoff + 1); pz = xs(I.xoff + 2); yaw = xs(I.xoff + 3); }
                else { px = I.pose[0]; py = I.pose[1]; pz = I.pose[2]; yaw = I.pose[3]; }
                float sy, cy;
                fsincos(yaw, &sy, &cy);
                const float* ob = P.obound[I.obj];
                ip(i, 0) = cy; ip(i, 1) = sy; ip(i, 2) = px; ip(i, 3) = py; ip(i, 4) = pz;
                ip(i, 5) = fmaf(cy, ob[0], fmaf(-sy, ob[1], px));
                ip(i, 6) = fmaf(sy, ob[0], fmaf(cy, ob[1], py));
                ip(i, 7) = pz + ob[2];
            }
            if (G && I.xoff >= 0)
                for (int k = 0; k < 6; ++k) iw(i, k) = 0.f;
        }
        if (G)
            for (int d = 0; d < D; ++d) gs(d) = 0.f;

        // ---- robot configurations ----
        for (int f = 0; f < P.n_fk; ++f) {
            const KFk K = P.fk[f];
            if (K.ghost) continue;
            TAMP_DCHECK(K.xoff >= 0 && K.xoff + TAMP_NJ <= D && K.part_begin + K.part_count <= kMaxPartners);
            float q[TAMP_NJ], sq[TAMP_NJ], cq[TAMP_NJ];
#pragma unroll
            for (int j = 0; j < TAMP_NJ; ++j) {
                q[j] = xs(K.xoff + j);
                fsincos(q[j], &sq[j], &cq[j]);
            }
            // forward: T_{j+1} = T_j F_{j+1} Rz(q_{j+1}) (base folded into F_1), tool T_8 = T_7 F_ee; T keeps its
            // rows 0-1 packed (M34P: FFMA2 compose, the scalar compose's values)
            // (joints 2..7 as modified-DH steps on the packed frame, dh_fwd; joint 1's F also carries the base)
            M34P T;
            {
                M34 A0;
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    const float* Fr = P.F[0] + 4 * i;
                    A0.r[3 * i] = fmaf(Fr[0], cq[0], Fr[1] * sq[0]);
                    A0.r[3 * i + 1] = fmaf(Fr[1], cq[0], -Fr[0] * sq[0]);
                    A0.r[3 * i + 2] = Fr[2];
                    A0.t[i] = Fr[3];
                }
                T = pack_m34(A0);
            }
#pragma unroll
            for (int j = 1; j < TAMP_NJ; ++j) dh_fwd(T, P.dh[j], cq[j], sq[j]);
            {
                M34 Fe;
                load_m34(Fe, P.F[kGroup - 1]);
                T = compose_p(T, Fe);
            }
            Wrench sfx;      // suffix wrench of the links >= the current one (about the world origin)
            sfx.zero();
            // Kin(q, o, g, p): FK(q) = T(p) T(g) at the tool frame
            if (K.term_kp >= 0 || K.term_kr >= 0) {
                const int ki = K.kin_inst;
                M34 Tg;
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    const int b = L.gT + 12 * K.kin_grasp + 4 * i;
                    Tg.r[3 * i] = col(b); Tg.r[3 * i + 1] = col(b + 1); Tg.r[3 * i + 2] = col(b + 2); Tg.t[i] = col(b + 3);
                }
                const float ipk[12] = {ip(ki, 0), 0.f, 0.f, ip(ki, 2), ip(ki, 1), 0.f, 0.f, ip(ki, 3), 0.f, 0.f, 0.f, ip(ki, 4)};
                const M34 Ts = compose_rz(ipk, Tg);   // T(p) T(g), T(p) = (Rz(yaw), t)
                const M34 Tu = unpack_m34(T);
                const float dx = Tu.t[0] - Ts.t[0], dy = Tu.t[1] - Ts.t[1], dz = Tu.t[2] - Ts.t[2];
                const float epos = sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
                float Mm[9];
#pragma unroll
                for (int i = 0; i < 3; ++i)
#pragma unroll
                    for (int j = 0; j < 3; ++j)
                        Mm[3 * i + j] = fmaf(Tu.r[i], Ts.r[j], fmaf(Tu.r[3 + i], Ts.r[3 + j], Tu.r[6 + i] * Ts.r[6 + j]));
                const float wx = Mm[7] - Mm[5], wy = Mm[2] - Mm[6], wz = Mm[3] - Mm[1];
                const float wn = sqrtf(fmaf(wx, wx, fmaf(wy, wy, wz * wz)));
                const float erot = fatan2_pos(0.5f * wn, 0.5f * (Mm[0] + Mm[4] + Mm[8] - 1.f));
                if (K.term_kp >= 0) serial_term<M>(P, A, sink, K.term_kp, epos, active, p, s_counts);
                if (K.term_kr >= 0) serial_term<M>(P, A, sink, K.term_kr, erot, active, p, s_counts);
                if (G) {
                    Wrench tw;
                    tw.zero();
                    if (K.term_kp >= 0 && epos > 0.f) {
                        const float k = P.term_lam[K.term_kp] / epos;
                        const float fx = dx * k, fy = dy * k, fz = dz * k;
                        sfx.add_point(Tu.t[0], Tu.t[1], Tu.t[2], fx, fy, fz);
                        tw.add_point(Ts.t[0], Ts.t[1], Ts.t[2], -fx, -fy, -fz);
                    }
                    if (K.term_kr >= 0 && wn > 0.f) {
                        const float k = P.term_lam[K.term_kr] / wn;
                        const float ux = k * fmaf(Tu.r[0], wx, fmaf(Tu.r[1], wy, Tu.r[2] * wz));
                        const float uy = k * fmaf(Tu.r[3], wx, fmaf(Tu.r[4], wy, Tu.r[5] * wz));
                        const float uz = k * fmaf(Tu.r[6], wx, fmaf(Tu.r[7], wy, Tu.r[8] * wz));
                        sfx.m[0] -= ux; sfx.m[1] -= uy; sfx.m[2] -= uz;
                        tw.m[0] += ux; tw.m[1] += uy; tw.m[2] += uz;
                    }
                    if (P.inst[ki].xoff >= 0) add_iw(ki, tw);
                }
            }
            // joint limits: dist_from_bounds(q, lo, hi) (Listing 2)
            float jl = 0.f;
            if (K.term_jl >= 0) {
                float e2 = 0.f;
#pragma unroll
                for (int j = 0; j < TAMP_NJ; ++j) {
                    const float e = fmaxf(fmaxf(P.jlo[j] - q[j], q[j] - P.jhi[j]), 0.f);
                    e2 = fmaf(e, e, e2);
                }
                jl = sqrtf(e2);
                serial_term<M>(P, A, sink, K.term_jl, jl, active, p, s_counts);
            }
            // backward sweep over the links 8 -> 1: spheres of link l in T_l, suffix wrench, dJ/dq_l
            const float lam_cf = K.term_cf >= 0 ? P.term_lam[K.term_cf] : 0.f;
            float jcf = 0.f;
            // one box to test (the table): its data in registers for the whole configuration
            const bool one_obb = K.obb_mask != 0 && (K.obb_mask & (K.obb_mask - 1)) == 0;
            KObb B0;
            if (one_obb) B0 = P.obb[__ffs(K.obb_mask) - 1];
            // PP: the per-configuration values the unrolled sweep uses, pinned in registers (opaque copies: the
            // compiler would otherwise re-load them from the constant bank with a computed index at every link)
            bool pp_cf = false, pp_jl = false;
            float pp_lam_jl = 0.f;
            int pp_g = 0;
            if constexpr (PP) {
                pp_cf = opaque_int(K.term_cf >= 0 && one_obb) != 0;
                pp_jl = opaque_int(K.term_jl >= 0 && jl > 0.f) != 0;
                pp_lam_jl = opaque_f(K.term_jl >= 0 ? P.term_lam[K.term_jl] : 0.f);
                pp_g = opaque_int(L.g + K.xoff);   // (an offset: the accesses stay shared-memory ones)
                if (one_obb) {
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        B0.c[i] = opaque_f(B0.c[i]); B0.h[i] = opaque_f(B0.h[i]);
                        B0.lo[i] = opaque_f(B0.lo[i]); B0.hi[i] = opaque_f(B0.hi[i]);
                    }
                }
            }
            // PP: the sweep unrolled (per-link data as constant-bank operands), only the packed one-box path
#pragma unroll (PP ? kGroup : 1)
            for (int l = kGroup - 1; l >= 0; --l) {
                // link broad phase (conservative, results unchanged): the link's bounding sphere against the
                // boxes and the partner instances' bounding spheres; a link that reaches none of them has only
                // zero hinges and zero gradients, so its spheres are skipped
                bool near = PP ? (pp_cf && P.rsph_n[l] > 0) : (K.term_cf >= 0 && P.rsph_n[l] > 0);
                if (PP) {
                    if (TAMP_SERIAL_LINK_BROAD && near) {
                        const float* lb = P.lbound[l];
                        float bx, by, bz;
                        xform_p(T, lb[0], lb[1], lb[2], bx, by, bz);
                        near = obb_within<true>(bx, by, bz, lb[3] + P.eta + kLinkMargin, B0);
                    }
                } else if (near) {
                    const float* lb = P.lbound[l];
                    float bx, by, bz;
                    xform_p(T, lb[0], lb[1], lb[2], bx, by, bz);
                    const float br = lb[3] + P.eta + kLinkMargin;
                    near = false;
                    if (one_obb) {
                        near = obb_within(bx, by, bz, br, B0);
                    } else {
                        for (int b = 0; b < P.n_obb; ++b)
                            if ((K.obb_mask >> b) & 1) near = near || obb_within(bx, by, bz, br, P.obb[b]);
                    }
                    for (int pi = 0; pi < K.part_count && !near; ++pi) {
                        const int ii = P.partners[K.part_begin + pi];
                        const float dx = bx - ip(ii, 5), dy = by - ip(ii, 6), dz = bz - ip(ii, 7);
                        const float R = br + P.obound[P.inst[ii].obj][3];
                        near = fmaf(-R, R, fmaf(dx, dx, fmaf(dy, dy, dz * dz))) < 0.f;
                    }
                }
                if (near && (PP || (one_obb && K.part_count == 0))) {
                    // one box, no partner instances (pick-place): the exact reject test of all of the link's
                    // spheres first (straight-line code, independent chains), hinges and gradients only for those
                    // that reach the box -- the others add exact zeros, so the result is unchanged
                    // (spheres in packed pairs: FFMA2 transforms and reject tests, the scalar code's values)
                    const int ns = P.rsph_n[l];
                    float wq[TAMP_MAX_SPHERES_PER_LINK][3], rq[TAMP_MAX_SPHERES_PER_LINK];
                    bool hit[TAMP_MAX_SPHERES_PER_LINK];
                    const float* cs = s_rsoa[l];
#pragma unroll
                    for (int kp = 0; kp < TAMP_MAX_SPHERES_PER_LINK / 2; ++kp) {
                        const F2 cx = *reinterpret_cast<const F2*>(cs + 2 * kp);
                        const F2 cy = *reinterpret_cast<const F2*>(cs + 4 + 2 * kp);
                        const F2 cz = *reinterpret_cast<const F2*>(cs + 8 + 2 * kp);
                        const F2 cr = *reinterpret_cast<const F2*>(cs + 12 + 2 * kp);
                        const F2 wx = fma2(bc(T.r(0, 0)), cx, fma2(bc(T.r(0, 1)), cy, fma2(bc(T.r(0, 2)), cz, bc(T.t(0)))));
                        const F2 wy = fma2(bc(T.r(1, 0)), cx, fma2(bc(T.r(1, 1)), cy, fma2(bc(T.r(1, 2)), cz, bc(T.t(1)))));
                        const F2 wz = fma2(bc(T.r(2, 0)), cx, fma2(bc(T.r(2, 1)), cy, fma2(bc(T.r(2, 2)), cz, bc(T.t(2)))));
                        bool h0, h1;
                        if (TAMP_BOX_CORNER && (PP || B0.aligned)) {
                            obb_reach_corner_pair(wx, wy, wz, cr, B0, h0, h1);
                        } else {
                            F2 px, py, pz;
                            obb_offsets_pair(wx, wy, wz, B0, px, py, pz);
                            obb_reach_pair(px, py, pz, cr, B0, h0, h1);
                        }
                        const int k = 2 * kp;
                        wq[k][0] = lo(wx); wq[k][1] = lo(wy); wq[k][2] = lo(wz); rq[k] = lo(cr);
                        wq[k + 1][0] = hi(wx); wq[k + 1][1] = hi(wy); wq[k + 1][2] = hi(wz); rq[k + 1] = hi(cr);
                        hit[k] = k < ns && h0;
                        hit[k + 1] = k + 1 < ns && h1;
                    }
                    // the exact hinges of the spheres that reach the box, in ascending sphere order (the same sums as
                    // one unrolled block per sphere): one rolled copy of the rare path per link, its operands
                    // selected from registers (a small kernel body: the link sweep is unrolled)
                    unsigned hm = 0;
#pragma unroll
                    for (int k = 0; k < TAMP_MAX_SPHERES_PER_LINK; ++k) hm |= hit[k] ? 1u << k : 0u;
#pragma unroll 1
                    while (hm) {
                        const int k = __ffs(hm) - 1;
                        hm &= hm - 1;
                        float x = wq[0][0], y = wq[0][1], z = wq[0][2], r = rq[0];
#pragma unroll
                        for (int u = 1; u < TAMP_MAX_SPHERES_PER_LINK; ++u)
                            if (k == u) { x = wq[u][0]; y = wq[u][1]; z = wq[u][2]; r = rq[u]; }
                        float g[3] = {0.f, 0.f, 0.f};
                        jcf += sphere_obb<G, PP>(x, y, z, r, B0, lam_cf, g[0], g[1], g[2], smooth);
                        if (G) sfx.add_point(x, y, z, g[0], g[1], g[2]);
                    }
                } else if (!PP && near) {
                    for (int k = 0; k < P.rsph_n[l]; ++k) {
                        const float4 c4 = s_rsph[l][k];
                        float wx, wy, wz;
                        xform_p(T, c4.x, c4.y, c4.z, wx, wy, wz);
                        const float rr = c4.w;
                        float g[3] = {0.f, 0.f, 0.f};
                        if (one_obb) {
                            bool near = true;
                            if (B0.rad < kBroadMaxRad) {
                                const float dx = wx - B0.c[0], dy = wy - B0.c[1], dz = wz - B0.c[2];
                                const float R = rr + B0.rad;
                                near = fmaf(-R, R, fmaf(dx, dx, fmaf(dy, dy, dz * dz))) < 0.f;
                            }
                            if (near) jcf += sphere_obb<G>(wx, wy, wz, rr, B0, lam_cf, g[0], g[1], g[2], smooth);
                        } else {
                            jcf += sphere_vs_obbs(wx, wy, wz, rr, K.obb_mask, lam_cf, g);
                        }
                        for (int pi = 0; pi < K.part_count; ++pi) {
                            const int ii = P.partners[K.part_begin + pi];
                            Wrench pw;
                            pw.zero();
                            jcf += sphere_vs_inst(wx, wy, wz, rr, ii, lam_cf, g, pw);
                            if (G && P.inst[ii].xoff >= 0 && pw.nonzero()) add_iw(ii, pw);
                        }
                        if (G) sfx.add_point(wx, wy, wz, g[0], g[1], g[2]);
                    }
                }
                if (l < TAMP_NJ) {     // joint l+1 rotates frame l+1 (= T here) about its z axis
                    if (G) {
                        const float zx = T.r(0, 2), zy = T.r(1, 2), zz = T.r(2, 2);
                        const float ox = T.t(0), oy = T.t(1), oz = T.t(2);
                        const float mx = sfx.m[0] - (oy * sfx.f[2] - oz * sfx.f[1]);
                        const float my = sfx.m[1] - (oz * sfx.f[0] - ox * sfx.f[2]);
                        const float mz = sfx.m[2] - (ox * sfx.f[1] - oy * sfx.f[0]);
                        float dq = fmaf(zx, mx, fmaf(zy, my, zz * mz));
                        if (PP) {
                            if (pp_jl) {
                                const float ql = q[l];
                                const float e = fmaxf(fmaxf(P.jlo[l] - ql, ql - P.jhi[l]), 0.f);
                                if (e > 0.f) dq += pp_lam_jl * (ql > P.jhi[l] ? e : -e) / jl;
                            }
                            col(pp_g + l) += dq;
                        } else if (K.term_jl >= 0 && jl > 0.f) {
                            const float ql = xs(K.xoff + l);
                            const float e = fmaxf(fmaxf(P.jlo[l] - ql, ql - P.jhi[l]), 0.f);
                            if (e > 0.f) dq += P.term_lam[K.term_jl] * (ql > P.jhi[l] ? e : -e) / jl;
                        }
                        if (!PP) gs(K.xoff + l) += dq;
                    }
                }
                if (l > 0) {           // T_{l} -> T_{l-1}: right-multiply by (F_l Rz(q_l))^-1 = Rz(-q_l) F_l^-1
                    if (l < TAMP_NJ) {   // a modified-DH joint (dh_bwd); PP: the forward pass's sin / cos
                        float sl, cl;
                        if constexpr (PP) { sl = sq[l]; cl = cq[l]; }
                        else fsincos(xs(K.xoff + l), &sl, &cl);
                        dh_bwd(T, P.dh[l], cl, sl);
                    } else {             // the tool frame
                        M34 Fi;
                        load_m34(Fi, P.Finv[l]);
                        T = compose_p(T, Fi);
                    }
                }
            }
            if (K.term_cf >= 0) serial_term<M>(P, A, sink, K.term_cf, jcf, active, p, s_counts);
            // block-synchronous configurations: every warp of the block executes the same (large) code region at
            // a time and the instruction cache is shared (the kernel body is ~100 KB of SASS)
            if (A.bsync && (!PP || TAMP_SERIAL_CONF_BARRIER)) __syncthreads();
        }

        // ---- StablePlace / press contact / CFreePlace per Place or press action ----
        for (int pl = 0; pl < P.n_place; ++pl) {
            const KPlace& Q = P.place[pl];
            const int ii = Q.inst;
            const KInst& I = P.inst[ii];
            const KSurface& Sf = P.surf[Q.surface];
            const int obj = I.obj, no = P.osph_n[obj];
            const IPose qi = ipose(ii);
            Wrench own;
            own.zero();
            {   // support |z_bottom - z_top|
                const float pz = ip(ii, 4);
                const float e = fabsf(pz - Sf.frame[2]);
                serial_term<M>(P, A, sink, Q.term_ss, e, active, p, s_counts);
                if (G && e > 0.f) own.add_point(ip(ii, 2), ip(ii, 3), pz, 0.f, 0.f, P.term_lam[Q.term_ss] * (pz > Sf.frame[2] ? 1.f : -1.f));
            }
            const float sy = Sf.sy, cy = Sf.cy;
            if (Q.term_sc >= 0) {   // containment: sum over spheres of dist_from_bounds(xy, lo + r, hi - r)
                float e = 0.f;
                for (int k = 0; k < no; ++k) {
                    const float4 c = inst_sphere(qi, obj, k);
                    const float rx = c.x - Sf.frame[0], ry = c.y - Sf.frame[1];
                    const float lx = fmaf(cy, rx, sy * ry), ly = fmaf(-sy, rx, cy * ry);
                    const float lox = Sf.lo[0] + c.w, hix = Sf.hi[0] - c.w;
                    const float loy = Sf.lo[1] + c.w, hiy = Sf.hi[1] - c.w;
                    const float ex = fmaxf(fmaxf(lox - lx, lx - hix), 0.f);
                    const float ey = fmaxf(fmaxf(loy - ly, ly - hiy), 0.f);
                    const float eu = sqrtf(fmaf(ex, ex, ey * ey));
                    e += eu;
                    if (G && eu > 0.f) {
                        const float kk = P.term_lam[Q.term_sc] / eu;
                        const float glx = (lx > hix ? ex : (lx < lox ? -ex : 0.f)) * kk;
                        const float gly = (ly > hiy ? ey : (ly < loy ? -ey : 0.f)) * kk;
                        own.add_point(c.x, c.y, c.z, fmaf(cy, glx, -sy * gly), fmaf(sy, glx, cy * gly), 0.f);
                    }
                }
                serial_term<M>(P, A, sink, Q.term_sc, e, active, p, s_counts);
            }
            if (Q.term_pc >= 0) {   // press contact: min over spheres of dist_from_bounds(xy, lo, hi)
                float emin = kFar, gx = 0.f, gy = 0.f, cx = 0.f, cyy = 0.f, cz = 0.f;
                for (int k = 0; k < no; ++k) {
                    const float4 c = inst_sphere(qi, obj, k);
                    const float rx = c.x - Sf.frame[0], ry = c.y - Sf.frame[1];
                    const float lx = fmaf(cy, rx, sy * ry), ly = fmaf(-sy, rx, cy * ry);
                    const float ex = fmaxf(fmaxf(Sf.lo[0] - lx, lx - Sf.hi[0]), 0.f);
                    const float ey = fmaxf(fmaxf(Sf.lo[1] - ly, ly - Sf.hi[1]), 0.f);
                    const float eu = sqrtf(fmaf(ex, ex, ey * ey));
                    if (eu < emin) {
                        emin = eu;
                        gx = eu > 0.f ? (lx > Sf.hi[0] ? ex : (lx < Sf.lo[0] ? -ex : 0.f)) / eu : 0.f;
                        gy = eu > 0.f ? (ly > Sf.hi[1] ? ey : (ly < Sf.lo[1] ? -ey : 0.f)) / eu : 0.f;
                        cx = c.x; cyy = c.y; cz = c.z;
                    }
                }
                serial_term<M>(P, A, sink, Q.term_pc, emin, active, p, s_counts);
                if (G && emin > 0.f) {
                    const float lam = P.term_lam[Q.term_pc];
                    own.add_point(cx, cyy, cz, lam * fmaf(cy, gx, -sy * gy), lam * fmaf(sy, gx, cy * gy), 0.f);
                }
            }
            if (Q.term_cp >= 0) {   // CFreePlace: the object's spheres vs OBBs (support excluded) and other objects
                const float lam_cp = P.term_lam[Q.term_cp];
                float jcp = 0.f;
                // no box besides the support and no partner (config 1): every hinge is zero -- nothing to test
                const int ncp = (Q.obb_mask || Q.part_count) ? no : 0;
                for (int k = 0; k < ncp; ++k) {
                    const float4 c = inst_sphere(qi, obj, k);
                    const float rr = c.w + P.eta;
                    float g[3] = {0.f, 0.f, 0.f};
                    if (Q.obb_mask) jcp += sphere_vs_obbs(c.x, c.y, c.z, rr, Q.obb_mask, lam_cp, g);
                    for (int pi = 0; pi < Q.part_count; ++pi) {
                        const int jj = P.partners[Q.part_begin + pi];
                        Wrench pw;
                        pw.zero();
                        jcp += sphere_vs_inst(c.x, c.y, c.z, rr, jj, lam_cp, g, pw);
                        if (G && P.inst[jj].xoff >= 0 && pw.nonzero()) add_iw(jj, pw);
                    }
                    if (G) own.add_point(c.x, c.y, c.z, g[0], g[1], g[2]);
                }
                serial_term<M>(P, A, sink, Q.term_cp, jcp, active, p, s_counts);
            }
            if (G && I.xoff >= 0) add_iw(ii, own);
            if (A.bsync) __syncthreads();
        }

        // ---- soft costs (Eq. 2 second sum) ----
        if (P.n_goal > 1) {   // MinimizeObjDist (Listing 2 obj_dist)
            for (int a = 0; a < P.n_goal; ++a)
                for (int b = a + 1; b < P.n_goal; ++b) {
                    const int ia = P.goal_inst[a], ib = P.goal_inst[b];
                    const float ax = ip(ia, 2), ay = ip(ia, 3), az = ip(ia, 4);
                    const float bx = ip(ib, 2), by = ip(ib, 3), bz = ip(ib, 4);
                    const float dx = ax - bx, dy = ay - by, dz = az - bz;
                    const float d = sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
                    soft = fmaf(P.lam_goal, d, soft);
                    if (G && d > 0.f) {
                        const float k = P.lam_goal / d;
                        Wrench w;
                        if (P.inst[ia].xoff >= 0) { w.zero(); w.add_point(ax, ay, az, dx * k, dy * k, dz * k); add_iw(ia, w); }
                        if (P.inst[ib].xoff >= 0) { w.zero(); w.add_point(bx, by, bz, -dx * k, -dy * k, -dz * k); add_iw(ib, w); }
                    }
                }
        }
        for (int tr = 0; tr < P.n_traj; ++tr) {   // TrajLength(tau) = sum_j ||k_{j+1} - k_j||
            const KTraj& Tj = P.traj[tr];
            const int nseg = Tj.n_knots + 1;
            auto xoff_of = [&](int j) -> int {
                if (j == 0) return Tj.q1_xoff;
                if (j == nseg) return Tj.q2_xoff;
                return Tj.knot_xoff + 7 * (j - 1);
            };
            auto val = [&](int j, int jt) -> float {
                const int o = xoff_of(j);
                if (o >= 0) return xs(o + jt);
                return P.const_conf[j == 0 ? Tj.q1_const : Tj.q2_const][jt];
            };
            for (int j = 0; j < nseg; ++j) {
                float dl[TAMP_NJ], s2 = 0.f;
#pragma unroll
                for (int jt = 0; jt < TAMP_NJ; ++jt) {
                    dl[jt] = val(j + 1, jt) - val(j, jt);
                    s2 = fmaf(dl[jt], dl[jt], s2);
                }
                const float len = sqrtf(s2);
                soft = fmaf(P.lam_traj, len, soft);
                if (G && len > 0.f) {
                    const int o1 = xoff_of(j + 1), o0 = xoff_of(j);
#pragma unroll
                    for (int jt = 0; jt < TAMP_NJ; ++jt) {
                        const float g = P.lam_traj * dl[jt] / len;
                        if (o1 >= 0) gs(o1 + jt) += g;
                        if (o0 >= 0) gs(o0 + jt) -= g;
                    }
                }
            }
        }
        const float Jtot = sink.J + soft;

        // ---- instance wrenches -> placement gradients: dJ/dt = F, dJ/dyaw = z . (M - t x F) ----
        if (G)
            for (int i = 0; i < P.n_inst; ++i) {
                const KInst& I = P.inst[i];
                if (I.xoff < 0) continue;
                gs(I.xoff) += iw(i, 0);
                gs(I.xoff + 1) += iw(i, 1);
                gs(I.xoff + 2) += iw(i, 2);
                gs(I.xoff + 3) += iw(i, 5) - (xs(I.xoff) * iw(i, 1) - xs(I.xoff + 1) * iw(i, 0));
            }

        if (M == MODE_EVAL) {
            if (active) {
                if (A.out_J) A.out_J[p] = Jtot;
                if (A.out_soft) A.out_soft[p] = soft;
                if (A.out_grad) for (int d = 0; d < D; ++d) A.out_grad[p * D + d] = gs(d);
            }
        } else if (M == MODE_CHECK) {
            const bool inv = invalid || !isfinite(Jtot);
            const int cls = inv ? 2 : (sink.sat ? 0 : 1);
            if (active) {
                A.out_cls[p] = (uint8_t)cls;
                A.out_cost[p] = cls == 0 ? soft : (cls == 1 ? Jtot : 0.f);
            }
            const unsigned b0 = __ballot_sync(FULL, active && cls == 0), b2 = __ballot_sync(FULL, active && cls == 2);
            if ((tid & 31) == 0) {
                if (b0) atomicAdd(&s_counts[P.n_terms], __popc(b0));
                if (b2) atomicAdd(&s_counts[P.n_terms + 1], __popc(b2));
            }
        } else {
            // ---- Adam (Kingma & Ba) with grad scale 1/N (Eq. 4) + projection (L11) ----
            // non-finite cost or gradient: g * 0 is 0 for finite g and NaN for an infinite or NaN one, so the sum
            // is 0 exactly when every entry is finite (one FFMA per coordinate)
            float nf = fmaf(Jtot, 0.f, 0.f);
            for (int d = 0; d < D; ++d) nf = fmaf(gs(d), 0.f, nf);
            invalid = invalid || !(nf == 0.f);
            const float rbc1 = A.rbc1[it];
            const float rbc2 = A.rbc2[it];
            if (!invalid && active) {
                // moments in the 32-particle tile layout: a warp's accesses to coordinate d are one 128-byte line;
                // loaded in batches of kB coordinates (one L2 latency per batch)
                float* const mt = A.m + mv_w32_index(pid, 0, D);
                float* const vt = A.v + mv_w32_index(pid, 0, D);
                constexpr int kB = TAMP_SERIAL_ADAM_BATCH;
                for (int d0 = 0; d0 < D; d0 += kB) {
                    float mo[kB], vo[kB];
#pragma unroll
                    for (int u = 0; u < kB; ++u) {
                        mo[u] = d0 + u < D ? mt[(d0 + u) * 32] : 0.f;
                        vo[u] = d0 + u < D ? vt[(d0 + u) * 32] : 0.f;
                    }
#pragma unroll
                    for (int u = 0; u < kB; ++u) {
                        const int d = d0 + u;
                        if (d >= D) break;
                        const float g = gs(d) * P.grad_scale;
                        const float mm = fmaf(P.beta1, mo[u], (1.f - P.beta1) * g);
                        const float vv = fmaf(P.beta2, vo[u], (1.f - P.beta2) * g * g);
                        mt[d * 32] = mm;
                        vt[d * 32] = vv;
                        const float mh = mm * rbc1;
                        const float vh = vv * rbc2;
                        // MUFU square root and reciprocal (flush-to-zero forms: no denormal rescaling around them)
                        const float xn = xs(d) - s_lr[d] * mh * rcp_approx(sqrt_approx(vh) + P.adam_eps);
                        xs(d) = fminf(fmaxf(xn, s_lr[D + d]), s_lr[2 * D + d]);
                    }
                }
            }
        }
    };
    for (int it = 0; it < n_iter; ++it) iteration(std::integral_constant<int, MODE>{}, it);
    if constexpr (MODE == MODE_OPT) {
        if (A.check_after) {            // Eq. 3 check of the final state in the same launch
            __syncthreads();
            iteration(std::integral_constant<int, MODE_CHECK>{}, n_iter);
        }
    }

    if (MODE == MODE_OPT) {
        if (active) A.invalid[p] = invalid ? 1 : 0;
        __syncthreads();
        store_rows(A.x, D, L.x);
    }
    if (MODE == MODE_CHECK || (MODE == MODE_OPT && A.check_after)) {
        __syncthreads();
        for (int i = tid; i < P.n_terms + 2; i += NT)
            if (s_counts[i]) atomicAdd(&A.out_counts[i], s_counts[i]);
    }
}

}  // namespace tamp
