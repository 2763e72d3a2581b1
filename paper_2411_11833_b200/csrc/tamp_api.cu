// tamp_api.cu -- host side of libtamp: descriptor validation, skeleton -> CSP compiler, workspace,
// and the extern "C" entry points declared in include/tamp.h.
//
// The compiler follows Listing 1 in deferred-motion mode plus knots for
// motions that carry a trajectory variable, simulating the symbolic state along the
// skeleton (which object is where / held) to decide which collision pairs each term checks
// (SURVEY §8(c) L3).  Canonical term order (shared contract with the oracle):
//   MoveFree/MoveHold with K knots: per knot  JL, CF
//   Pick(o, g, p, q):                          JL(q), CF(q) [o excluded], KP(q), KR(q)
//   Place(o, g, p, s, q):                      JL(q), CF(q) [held o excluded], KP(q), KR(q), SS(p), SC(p), CP(p)
#include <cuda_runtime.h>

#include <algorithm>
#include <tuple>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tamp.h"
#include "tamp_program.h"
#include "particle_serial.cuh"

namespace tamp {
cudaError_t launch_particle(int mode, int gs, int bsync, int threads, const KProgram& P, const KArgs& A, size_t smem,
                            cudaStream_t st);
cudaError_t launch_sample(const KSampleProgram& SP, float* x, float* grasp, int64_t n, int64_t gofs, uint64_t seed,
                          cudaStream_t st);
cudaError_t launch_ik(const KProgram& P, const KSampleProgram& SP, float* x, const float* grasp, int64_t n, int64_t gofs,
                      uint64_t seed, int iters, float damping, int n_seeds, int32_t* lists, int32_t* list_n,
                      float* best, cudaStream_t st);
int particle_kernel_regs(int gs, int threads);
int serial_kernel_regs(bool pp);
#ifndef TAMP_SERIAL_PP
#define TAMP_SERIAL_PP 1
#endif
cudaError_t launch_topk(unsigned long long* ka, int32_t* pa, unsigned long long* kb, int32_t* pb, int64_t n, int k,
                        cudaStream_t st, unsigned long long** kres, int32_t** pres);
cudaError_t launch_make_keys(const uint8_t* cls, const float* cost, int64_t n, int64_t gofs, unsigned long long* keys,
                             int32_t* pay, cudaStream_t st);
cudaError_t launch_record_keys(const float* rec, int32_t n, int32_t width, unsigned long long* keys, int32_t* pay,
                               cudaStream_t st);
cudaError_t launch_gather_particles(const int32_t* pay, const unsigned long long* keys, int k, const float* x,
                                    const float* cost, int D, int64_t gofs, float* rec, cudaStream_t st);
cudaError_t launch_mv_layout(const float* src, float* dst, int64_t n, int D, int to_w32, cudaStream_t st);
cudaError_t launch_gather_records(const int32_t* pay, int k, const float* rin, int width, float* rout, cudaStream_t st);
uint64_t launch_count();
}  // namespace tamp

using namespace tamp;

static thread_local std::string g_err;

static tamp_status fail(tamp_status s, const std::string& msg) {
    g_err = msg;
    return s;
}

static tamp_status cuda_fail(cudaError_t e, const char* where) {
    return fail(TAMP_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CUDA_TRY(call, where)                          \
    do {                                               \
        cudaError_t e_ = (call);                       \
        if (e_ != cudaSuccess) return cuda_fail(e_, where); \
    } while (0)

struct tamp_ctx {
    int device = 0;
    int64_t n = 0, gofs = 0, nglob = 0;
    KProgram P;
    KSampleProgram SP;
    char* base = nullptr;
    size_t ws_bytes = 0;
    // workspace offsets
    size_t o_x, o_m, o_v, o_grasp, o_inv, o_cls, o_cost, o_ka, o_kb, o_pa, o_pb, o_coords, o_counts, o_stage, o_iklist, o_ikn, o_ikbest, total;
    int64_t n_keys = 0;
    // shared-memory layout of the particle kernel (floats per particle)
    int stride, off_g, off_inst, off_gT, off_gTi, off_rsw, const_floats, fk_off, pw_off, n_pw;
    size_t smem = 0;
    int gs = 8;                  // lanes per particle in the particle kernel
    int ik_iters = 0;            // conditional IK sampler iterations
    float ik_damping = 0.1f;
    int ik_seeds = 1;            // IK restarts per conf (1, 2, 4, 8)
    int threads = 128;           // particle-kernel block size
    int bsync = 2;               // block-synchronisation level of the particle kernel (0..2)
    int stride_bytes = 0;
    int32_t t = 0;
    bool ready = false;
    bool checked = false;        // cls / cost / counts are those of the current state (no step since)
    int32_t term_kind[TAMP_MAX_TERMS];
    int32_t term_action[TAMP_MAX_TERMS];
    std::vector<float> coords;   // lr | lo | hi, uploaded (stream-ordered) by the first sample / set_state
    bool coords_on_device = false;
    int64_t pairs_sb = 0, pairs_ss = 0;
    int32_t n_robot_spheres = 0;

    template <class T>
    T* at(size_t off) const { return reinterpret_cast<T*>(base + off); }
};

// ------------------------------------------------------------------------------------------------
// small double-precision transform helpers (host, compile time only)
// ------------------------------------------------------------------------------------------------
struct H34 {
    double r[9];
    double t[3];
};
static H34 h_ident() { H34 a{}; a.r[0] = a.r[4] = a.r[8] = 1.0; return a; }
static H34 h_mul(const H34& a, const H34& b) {
    H34 c{};
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j)
            c.r[3 * i + j] = a.r[3 * i] * b.r[j] + a.r[3 * i + 1] * b.r[3 + j] + a.r[3 * i + 2] * b.r[6 + j];
        c.t[i] = a.r[3 * i] * b.t[0] + a.r[3 * i + 1] * b.t[1] + a.r[3 * i + 2] * b.t[2] + a.t[i];
    }
    return c;
}
static H34 h_rx(double a) { H34 m = h_ident(); m.r[4] = cos(a); m.r[5] = -sin(a); m.r[7] = sin(a); m.r[8] = cos(a); return m; }
static H34 h_rz(double a) { H34 m = h_ident(); m.r[0] = cos(a); m.r[1] = -sin(a); m.r[3] = sin(a); m.r[4] = cos(a); return m; }
static H34 h_tr(double x, double y, double z) { H34 m = h_ident(); m.t[0] = x; m.t[1] = y; m.t[2] = z; return m; }
static H34 h_inv(const H34& a) {
    H34 o{};
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) o.r[3 * i + j] = a.r[3 * j + i];
    for (int i = 0; i < 3; ++i) o.t[i] = -(o.r[3 * i] * a.t[0] + o.r[3 * i + 1] * a.t[1] + o.r[3 * i + 2] * a.t[2]);
    return o;
}
static void h_store(const H34& a, float* o) {
    for (int i = 0; i < 3; ++i) {
        o[4 * i] = (float)a.r[3 * i]; o[4 * i + 1] = (float)a.r[3 * i + 1];
        o[4 * i + 2] = (float)a.r[3 * i + 2]; o[4 * i + 3] = (float)a.t[i];
    }
}

static size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

// ------------------------------------------------------------------------------------------------
// compiler
// ------------------------------------------------------------------------------------------------
struct Compiled {
    KProgram P;
    KSampleProgram SP;
    std::vector<float> lr, lo, hi;
    int32_t term_kind[TAMP_MAX_TERMS];
    int32_t term_action[TAMP_MAX_TERMS];
    int64_t pairs_sb = 0, pairs_ss = 0;
};

// collision pairs evaluated per particle-step (all pairs; the kernel's culling is an implementation detail)
static void count_pairs(const tamp_problem_desc& d, Compiled& C) {
    const KProgram& P = C.P;
    auto popc = [](uint32_t m) { int c = 0; while (m) { c += m & 1; m >>= 1; } return c; };
    int64_t sb = 0, ss = 0;
    for (int f = 0; f < P.n_fk; ++f) {
        const KFk& K = P.fk[f];
        if (K.term_cf < 0 || K.ghost) continue;
        int part_sph = 0;
        for (int i = 0; i < K.part_count; ++i) part_sph += P.osph_n[P.inst[P.partners[K.part_begin + i]].obj];
        const int nb = popc(K.obb_mask);
        sb += (int64_t)d.robot.n_spheres * nb;
        ss += (int64_t)d.robot.n_spheres * part_sph;
        if (K.held_grasp >= 0) { sb += (int64_t)P.osph_n[K.held_obj] * nb; ss += (int64_t)P.osph_n[K.held_obj] * part_sph; }
    }
    for (int q = 0; q < P.n_place; ++q) {
        const KPlace& Q = P.place[q];
        if (Q.term_cp < 0) continue;
        int part_sph = 0;
        for (int i = 0; i < Q.part_count; ++i) part_sph += P.osph_n[P.inst[P.partners[Q.part_begin + i]].obj];
        const int no = P.osph_n[P.inst[Q.inst].obj];
        sb += (int64_t)no * popc(Q.obb_mask);
        ss += (int64_t)no * part_sph;
    }
    C.pairs_sb = sb;
    C.pairs_ss = ss;
}

#define REQUIRE(cond, st, msg)                    \
    do {                                          \
        if (!(cond)) return fail(st, msg);        \
    } while (0)

// Every index the kernels dereference, checked against its array once per compile (defence in depth: the
// kernels do no bounds checks in the step loop, and compute-sanitizer is not available on the GPU pool).
static tamp_status check_program(const KProgram& P, const KSampleProgram& SP) {
    auto term_ok = [&](int t) { return t == -1 || (t >= 0 && t < P.n_terms); };
    auto conf_ok = [&](int xoff) { return xoff >= 0 && xoff + TAMP_NJ <= P.D; };
    auto inst_ok = [&](int i) { return i >= 0 && i < P.n_inst; };
    auto grasp_ok = [&](int g) { return g >= 0 && g < P.n_grasp; };
    auto partners_ok = [&](int b, int n) {
        if (b < 0 || n < 0 || b + n > kMaxPartners) return false;
        for (int k = 0; k < n; ++k) if (!inst_ok(P.partners[b + k])) return false;
        return true;
    };
    const uint32_t obb_all = (1u << P.n_obb) - 1u;
    REQUIRE(P.n_terms >= 0 && P.n_terms <= TAMP_MAX_TERMS && P.n_fk <= TAMP_MAX_FK && P.n_inst <= kMaxInst &&
            P.n_place <= kMaxPlace && P.n_traj <= kMaxTraj && P.D <= TAMP_MAX_D && P.n_grasp <= TAMP_MAX_GRASPS,
            TAMP_E_UNSUPPORTED, "internal: program sizes out of range");
    for (int f = 0; f < P.n_fk; ++f) {
        const KFk& K = P.fk[f];
        REQUIRE(conf_ok(K.xoff) && term_ok(K.term_jl) && term_ok(K.term_cf) && term_ok(K.term_kp) &&
                term_ok(K.term_kr) && term_ok(K.term_self) && (K.obb_mask & ~obb_all) == 0 &&
                partners_ok(K.part_begin, K.part_count), TAMP_E_INVALID, "internal: configuration entry out of range");
        if (K.term_kp >= 0 || K.term_kr >= 0)
            REQUIRE(inst_ok(K.kin_inst) && grasp_ok(K.kin_grasp), TAMP_E_INVALID, "internal: Kin target out of range");
        if (K.held_grasp >= 0)
            REQUIRE(grasp_ok(K.held_grasp) && K.held_obj >= 0 && K.held_obj < TAMP_MAX_OBJECTS, TAMP_E_INVALID,
                    "internal: held object out of range");
    }
    for (int i = 0; i < P.n_inst; ++i) {
        const KInst& I = P.inst[i];
        REQUIRE(I.obj >= 0 && I.obj < TAMP_MAX_OBJECTS && (I.xoff < 0 || I.xoff + 4 <= P.D), TAMP_E_INVALID,
                "internal: object instance out of range");
    }
    for (int q = 0; q < P.n_place; ++q) {
        const KPlace& Q = P.place[q];
        REQUIRE(inst_ok(Q.inst) && P.inst[Q.inst].xoff >= 0 && term_ok(Q.term_ss) && Q.term_ss >= 0 &&
                term_ok(Q.term_sc) && term_ok(Q.term_cp) && term_ok(Q.term_pc) && Q.surface >= 0 &&
                Q.surface < TAMP_MAX_SURFACES && (Q.obb_mask & ~obb_all) == 0 && partners_ok(Q.part_begin, Q.part_count),
                TAMP_E_INVALID, "internal: place / press entry out of range");
    }
    for (int t = 0; t < P.n_traj; ++t) {
        const KTraj& Tj = P.traj[t];
        REQUIRE((Tj.q1_xoff >= 0 ? conf_ok(Tj.q1_xoff) : (Tj.q1_const >= 0 && Tj.q1_const < kMaxConstConf)) &&
                (Tj.q2_xoff >= 0 ? conf_ok(Tj.q2_xoff) : (Tj.q2_const >= 0 && Tj.q2_const < kMaxConstConf)) &&
                Tj.n_knots >= 1 && Tj.knot_xoff >= 0 && Tj.knot_xoff + TAMP_NJ * Tj.n_knots <= P.D,
                TAMP_E_INVALID, "internal: trajectory entry out of range");
    }
    for (int k = 0; k < P.n_goal; ++k) REQUIRE(inst_ok(P.goal_inst[k]), TAMP_E_INVALID, "internal: goal out of range");
    for (int v = 0; v < SP.n_vars; ++v) {
        const KSVar& V = SP.v[v];
        if (V.kind == KS_GRASP) REQUIRE(grasp_ok(V.slot), TAMP_E_INVALID, "internal: sampler grasp slot out of range");
        else if (V.kind == KS_PLACEMENT) REQUIRE(V.xoff >= 0 && V.xoff + 4 <= P.D, TAMP_E_INVALID, "internal: sampler placement");
        else if (V.kind == KS_CONF) REQUIRE(conf_ok(V.xoff), TAMP_E_INVALID, "internal: sampler conf out of range");
        else REQUIRE(V.xoff >= 0 && V.xoff + TAMP_NJ * V.n_knots <= P.D, TAMP_E_INVALID, "internal: sampler knots");
    }
    return TAMP_OK;
}

static tamp_status compile(const tamp_problem_desc& d, int64_t n_global, Compiled& C) {
    std::memset(&C.P, 0, sizeof(C.P));
    std::memset(&C.SP, 0, sizeof(C.SP));
    KProgram& P = C.P;
    KSampleProgram& SP = C.SP;
    REQUIRE(d.abi_version == TAMP_ABI_VERSION, TAMP_E_INVALID, "abi_version mismatch");
    const tamp_robot_desc& R = d.robot;
    REQUIRE(d.n_obb >= 0 && d.n_obb <= TAMP_MAX_OBB, TAMP_E_UNSUPPORTED, "n_obb out of range");
    REQUIRE(d.n_objects >= 0 && d.n_objects <= TAMP_MAX_OBJECTS, TAMP_E_UNSUPPORTED, "n_objects out of range");
    REQUIRE(d.n_surfaces >= 0 && d.n_surfaces <= TAMP_MAX_SURFACES, TAMP_E_UNSUPPORTED, "n_surfaces out of range");
    REQUIRE(d.n_vars >= 0 && d.n_vars <= TAMP_MAX_VARS, TAMP_E_UNSUPPORTED, "n_vars out of range");
    REQUIRE(d.n_actions >= 0 && d.n_actions <= TAMP_MAX_ACTIONS, TAMP_E_UNSUPPORTED, "n_actions out of range");
    REQUIRE(d.n_goal >= 0 && d.n_goal <= TAMP_MAX_GOAL, TAMP_E_UNSUPPORTED, "n_goal out of range");
    REQUIRE(R.n_spheres >= 0 && R.n_spheres <= TAMP_MAX_ROBOT_SPHERES, TAMP_E_UNSUPPORTED, "robot n_spheres out of range");
    for (int j = 0; j < TAMP_NJ; ++j)
        REQUIRE(R.joint_lo[j] < R.joint_hi[j], TAMP_E_INVALID, "joint_lo must be < joint_hi (S:27)");
    for (int k = 0; k < TAMP_N_TERM_KINDS; ++k) {
        REQUIRE(d.lam[k] > 0.f && std::isfinite(d.lam[k]), TAMP_E_INVALID, "lambda must be > 0 (S:131)");
        REQUIRE(d.eps[k] >= 0.f && std::isfinite(d.eps[k]), TAMP_E_INVALID, "eps must be >= 0 (S:131)");
    }
    REQUIRE(d.eta >= 0.f, TAMP_E_INVALID, "eta must be >= 0");
    REQUIRE(d.beta1 >= 0.f && d.beta1 < 1.f && d.beta2 >= 0.f && d.beta2 < 1.f && d.adam_eps > 0.f, TAMP_E_INVALID,
            "Adam betas must be in [0,1), eps > 0");
    REQUIRE(d.lr_conf >= 0 && d.lr_pos >= 0 && d.lr_yaw >= 0 && d.lr_knot >= 0, TAMP_E_INVALID, "lr must be >= 0");
    REQUIRE(d.lam_goal >= 0 && d.lam_traj >= 0, TAMP_E_INVALID, "soft weights must be >= 0");

    // robot: fixed transforms (base folded into F_1) and per-link spheres
    {
        H34 T = h_mul(h_tr(R.base[0], R.base[1], R.base[2]), h_rz(R.base[3]));
        for (int j = 0; j < TAMP_NJ; ++j) {
            const double a = R.dh[j][0], dd = R.dh[j][1], al = R.dh[j][2];
            H34 F = h_mul(h_rx(al), h_tr(a, 0.0, dd));
            if (j == 0) F = h_mul(T, F);
            P.dh[j][0] = (float)a;
            P.dh[j][1] = (float)dd;
            P.dh[j][2] = (float)std::cos(al);
            P.dh[j][3] = (float)std::sin(al);
            h_store(F, P.F[j]);
            h_store(h_inv(F), P.Finv[j]);
            P.jlo[j] = R.joint_lo[j];
            P.jhi[j] = R.joint_hi[j];
            SP.jlo[j] = R.joint_lo[j];
            SP.jhi[j] = R.joint_hi[j];
        }
        H34 tool = h_mul(h_mul(h_tr(0, 0, R.flange_d), h_rz(R.tcp_yaw)), h_tr(0, 0, R.tcp_d));
        h_store(tool, P.F[kGroup - 1]);
        h_store(h_inv(tool), P.Finv[kGroup - 1]);
        int packed[TAMP_MAX_ROBOT_SPHERES];
        for (int s = 0; s < R.n_spheres; ++s) {
            const int l = R.sphere_link[s];
            REQUIRE(l >= 1 && l <= 8, TAMP_E_INVALID, "sphere_link must be in 1..8");
            REQUIRE(R.sphere[s][3] > 0.f, TAMP_E_INVALID, "robot sphere radius must be > 0 (S:36)");
            const int lane = l - 1;
            REQUIRE(P.rsph_n[lane] < TAMP_MAX_SPHERES_PER_LINK, TAMP_E_UNSUPPORTED, "more than 4 spheres on a link");
            for (int c = 0; c < 4; ++c) P.rsph[lane][P.rsph_n[lane]][c] = R.sphere[s][c];
            packed[s] = lane * TAMP_MAX_SPHERES_PER_LINK + P.rsph_n[lane];
            P.rsph_n[lane]++;
        }
        // link bounding spheres (self-collision broad phase)
        for (int l = 0; l < kGroup; ++l) {
            double c[3] = {0, 0, 0}, rad = 0;
            const int ns = P.rsph_n[l];
            for (int k = 0; k < ns; ++k)
                for (int a = 0; a < 3; ++a) c[a] += P.rsph[l][k][a] / ns;
            for (int k = 0; k < ns; ++k) {
                const double dx = P.rsph[l][k][0] - c[0], dy = P.rsph[l][k][1] - c[1], dz = P.rsph[l][k][2] - c[2];
                rad = std::max(rad, std::sqrt(dx * dx + dy * dy + dz * dz) + P.rsph[l][k][3]);
            }
            for (int a = 0; a < 3; ++a) P.lbound[l][a] = (float)c[a];
            P.lbound[l][3] = ns ? (float)(rad * (1.0 + 1e-5) + 1e-6) : 0.f;   // no spheres: no pairs either
        }
        // self-collision pairs in packed sphere ids
        if (d.self_collision) {
            P.has_self = 1;
            for (int i = 0; i < R.n_spheres; ++i)
                for (int j = 0; j < R.n_spheres; ++j) {
                    if (!((R.self_mask[i] >> j) & 1u)) continue;
                    REQUIRE(i != j && ((R.self_mask[j] >> i) & 1u), TAMP_E_INVALID, "self_mask must be symmetric, no diagonal");
                    P.self_mask[packed[i]] |= 1u << packed[j];
                }
        }
    }
    // world
    P.n_obb = d.n_obb;
    REQUIRE(d.n_obb <= 16, TAMP_E_UNSUPPORTED, "n_obb > 16");
    for (int b = 0; b < d.n_obb; ++b) {
        const tamp_obb_desc& o = d.obb[b];
        for (int k = 0; k < 3; ++k) REQUIRE(o.half[k] > 0.f, TAMP_E_INVALID, "OBB half extents must be > 0 (S:32)");
        KObb& B = P.obb[b];
        bool given = false;
        for (int k = 0; k < 9; ++k) given |= o.rot[k] != 0.f;
        double Rm[9];
        if (given) {            // full orientation: orthonormal, det +1
            for (int k = 0; k < 9; ++k) Rm[k] = o.rot[k];
            double err = 0.0;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) {
                    double d = 0.0;
                    for (int k = 0; k < 3; ++k) d += Rm[3 * k + i] * Rm[3 * k + j];
                    err = std::max(err, std::fabs(d - (i == j ? 1.0 : 0.0)));
                }
            const double det = Rm[0] * (Rm[4] * Rm[8] - Rm[5] * Rm[7]) - Rm[1] * (Rm[3] * Rm[8] - Rm[5] * Rm[6]) +
                               Rm[2] * (Rm[3] * Rm[7] - Rm[4] * Rm[6]);
            REQUIRE(err < 1e-4 && std::fabs(det - 1.0) < 1e-4, TAMP_E_INVALID, "OBB rot must be a rotation matrix");
        } else {                // Rz(yaw)
            const double c = cos((double)o.yaw), s = sin((double)o.yaw);
            const double Rz[9] = {c, -s, 0, s, c, 0, 0, 0, 1};
            for (int k = 0; k < 9; ++k) Rm[k] = Rz[k];
        }
        B.aligned = 1;
        for (int k = 0; k < 9; ++k) {
            B.R[k] = (float)Rm[k];
            B.aligned &= B.R[k] == ((k % 4 == 0) ? 1.f : 0.f);
        }
        for (int k = 0; k < 3; ++k) { B.c[k] = o.center[k]; B.h[k] = o.half[k]; }
        for (int k = 0; k < 3; ++k) {
            REQUIRE(std::fabs((double)o.center[k]) + o.half[k] <= kMaxCoord, TAMP_E_UNSUPPORTED,
                    "OBB extents beyond 100 m of the origin");
            B.lo[k] = std::nextafter((float)((double)B.c[k] - B.h[k] - kCornerSlack), -INFINITY);
            B.hi[k] = std::nextafter((float)((double)B.c[k] + B.h[k] + kCornerSlack), INFINITY);
        }
        B.rad = (float)(std::sqrt((double)o.half[0] * o.half[0] + (double)o.half[1] * o.half[1] +
                                  (double)o.half[2] * o.half[2]) * (1.0 + 1e-6));
    }
    const uint16_t all_obb = (uint16_t)((1u << d.n_obb) - 1u);
    for (int o = 0; o < d.n_objects; ++o) {
        const tamp_object_desc& ob = d.object[o];
        REQUIRE(ob.n_spheres >= 1 && ob.n_spheres <= TAMP_MAX_OBJ_SPHERES, TAMP_E_UNSUPPORTED,
                "object n_spheres must be in 1..8");
        P.osph_n[o] = ob.n_spheres;
        double ctr[3] = {0, 0, 0};
        for (int k = 0; k < ob.n_spheres; ++k) {
            REQUIRE(ob.sphere[k][3] > 0.f, TAMP_E_INVALID, "object sphere radius must be > 0 (S:36)");
            for (int c = 0; c < 4; ++c) P.osph[o][k][c] = ob.sphere[k][c];
            for (int c = 0; c < 3; ++c) ctr[c] += ob.sphere[k][c] / ob.n_spheres;
        }
        double rad = 0;   // bounding sphere (broad phase only: it never changes a cost, it skips far pairs)
        for (int k = 0; k < ob.n_spheres; ++k) {
            const double dx = ob.sphere[k][0] - ctr[0], dy = ob.sphere[k][1] - ctr[1], dz = ob.sphere[k][2] - ctr[2];
            rad = std::max(rad, std::sqrt(dx * dx + dy * dy + dz * dz) + ob.sphere[k][3]);
        }
        for (int c = 0; c < 3; ++c) P.obound[o][c] = (float)ctr[c];
        P.obound[o][3] = (float)(rad * (1.0 + 1e-5) + 1e-6);
    }
    for (int s = 0; s < d.n_surfaces; ++s) {
        const tamp_surface_desc& S = d.surface[s];
        REQUIRE(S.lo[0] <= S.hi[0] && S.lo[1] <= S.hi[1], TAMP_E_INVALID, "surface lo must be <= hi");
        REQUIRE(S.support_obb < d.n_obb && S.support_obj < d.n_objects, TAMP_E_INVALID, "surface support out of range");
        for (int k = 0; k < 4; ++k) P.surf[s].frame[k] = S.frame[k];
        P.surf[s].cy = (float)cos((double)S.frame[3]);
        P.surf[s].sy = (float)sin((double)S.frame[3]);
        for (int k = 0; k < 2; ++k) { P.surf[s].lo[k] = S.lo[k]; P.surf[s].hi[k] = S.hi[k]; }
    }

    // particle layout (free variables in declaration order; grasps frozen in their own array)
    std::vector<int> xoff(d.n_vars, -1), gslot(d.n_vars, -1), cconf(d.n_vars, -1), inst_of(d.n_vars, -1);
    int D = 0, G = 0, n_const = 0;
    for (int v = 0; v < d.n_vars; ++v) {
        const tamp_var_desc& V = d.var[v];
        REQUIRE(V.kind >= 0 && V.kind <= 3, TAMP_E_INVALID, "bad variable kind");
        if (V.kind == TAMP_VAR_GRASP) {
            REQUIRE(V.obj >= 0 && V.obj < d.n_objects, TAMP_E_INVALID, "grasp variable without object");
            REQUIRE(G < TAMP_MAX_GRASPS, TAMP_E_UNSUPPORTED, "too many grasps");
            gslot[v] = G++;
            continue;
        }
        if (V.is_const) {
            if (V.kind == TAMP_VAR_CONF) {
                REQUIRE(n_const < kMaxConstConf, TAMP_E_UNSUPPORTED, "too many constant confs");
                for (int j = 0; j < 7; ++j) { P.const_conf[n_const][j] = V.value[j]; SP.const_conf[n_const][j] = V.value[j]; }
                cconf[v] = n_const++;
            }
            REQUIRE(V.kind != TAMP_VAR_TRAJ, TAMP_E_UNSUPPORTED, "constant trajectories unsupported");
            continue;
        }
        xoff[v] = D;
        if (V.kind == TAMP_VAR_CONF) {
            for (int j = 0; j < 7; ++j) { C.lr.push_back(d.lr_conf); C.lo.push_back(R.joint_lo[j]); C.hi.push_back(R.joint_hi[j]); }
            D += 7;
        } else if (V.kind == TAMP_VAR_PLACEMENT) {
            REQUIRE(V.obj >= 0 && V.obj < d.n_objects, TAMP_E_INVALID, "placement variable without object");
            REQUIRE(V.surface >= 0 && V.surface < d.n_surfaces, TAMP_E_INVALID, "placement variable without surface");
            for (int j = 0; j < 4; ++j) {
                REQUIRE(V.lo[j] <= V.hi[j], TAMP_E_INVALID, "placement bounds lo must be <= hi");
                C.lr.push_back(j < 3 ? d.lr_pos : d.lr_yaw); C.lo.push_back(V.lo[j]); C.hi.push_back(V.hi[j]);
            }
            D += 4;
        } else {   // TRAJ
            REQUIRE(V.n_knots >= 0 && V.n_knots <= TAMP_MAX_KNOTS, TAMP_E_UNSUPPORTED, "n_knots out of range");
            for (int k = 0; k < V.n_knots; ++k)
                for (int j = 0; j < 7; ++j) { C.lr.push_back(d.lr_knot); C.lo.push_back(R.joint_lo[j]); C.hi.push_back(R.joint_hi[j]); }
            D += 7 * V.n_knots;
        }
        REQUIRE(D <= TAMP_MAX_D, TAMP_E_UNSUPPORTED, "D exceeds TAMP_MAX_D");
    }
    P.D = SP.D = D;
    P.n_grasp = SP.n_grasp = G;

    // object instances: every placement variable (constant initial poses and Place targets)
    int n_inst = 0;
    std::vector<int> init_inst(d.n_objects, -1);
    for (int v = 0; v < d.n_vars; ++v) {
        const tamp_var_desc& V = d.var[v];
        if (V.kind != TAMP_VAR_PLACEMENT) continue;
        REQUIRE(V.obj >= 0 && V.obj < d.n_objects, TAMP_E_INVALID, "placement variable without object");
        REQUIRE(n_inst < kMaxInst, TAMP_E_UNSUPPORTED, "too many object instances");
        KInst& I = P.inst[n_inst];
        I.obj = (int16_t)V.obj;
        I.xoff = (int16_t)(V.is_const ? -1 : xoff[v]);
        int slot = 0;
        for (int j = 0; j < n_inst; ++j) slot += (P.inst[j].xoff < 0) == (I.xoff < 0);
        I.slot = (int16_t)slot;
        for (int k = 0; k < 4; ++k) I.pose[k] = V.is_const ? V.value[k] : 0.f;
        if (V.is_const && init_inst[V.obj] < 0) init_inst[V.obj] = n_inst;
        inst_of[v] = n_inst++;
    }
    P.n_inst = n_inst;

    // symbolic simulation along the skeleton.  An object without a constant initial placement is virtual
    // (the PressButton fingertip): never in the scene.
    std::vector<int> pose(d.n_objects);   // object -> instance, -1 = held, -2 = virtual (absent)
    for (int o = 0; o < d.n_objects; ++o) pose[o] = init_inst[o] >= 0 ? init_inst[o] : -2;
    int held = -1;
    int n_terms = 0, n_fk = 0, n_place = 0, n_traj = 0, n_part = 0;
    int cur_action = -1;
    auto add_term = [&](int kind) -> int16_t {
        if (n_terms >= TAMP_MAX_TERMS) return -1;
        P.term_lam[n_terms] = d.lam[kind];
        P.term_eps[n_terms] = d.eps[kind];
        C.term_kind[n_terms] = kind;
        C.term_action[n_terms] = cur_action;
        return (int16_t)n_terms++;
    };
    auto add_partners = [&](int skip_a, int skip_b, int16_t& begin, int16_t& count) -> bool {
        begin = (int16_t)n_part;
        count = 0;
        for (int o = 0; o < d.n_objects; ++o) {
            if (pose[o] < 0 || o == skip_a || o == skip_b) continue;
            if (n_part >= kMaxPartners) return false;
            P.partners[n_part++] = (int16_t)pose[o];
            count++;
        }
        return true;
    };
    auto conf_ok = [&](int v) { return v >= 0 && v < d.n_vars && d.var[v].kind == TAMP_VAR_CONF; };
    for (int ai = 0; ai < d.n_actions; ++ai) {
        const tamp_action_desc& a = d.action[ai];
        cur_action = ai;
        if (a.kind == TAMP_MOVE_FREE || a.kind == TAMP_MOVE_HOLD) {
            REQUIRE(conf_ok(a.q1) && conf_ok(a.q2), TAMP_E_INVALID, "motion endpoints must be conf variables");
            if (a.kind == TAMP_MOVE_HOLD) REQUIRE(held == a.obj && a.obj >= 0, TAMP_E_INVALID, "MoveHold: object not held");
            if (a.traj < 0) continue;
            REQUIRE(a.traj < d.n_vars && d.var[a.traj].kind == TAMP_VAR_TRAJ && !d.var[a.traj].is_const, TAMP_E_INVALID,
                    "motion traj must be a free traj variable");
            const int K = d.var[a.traj].n_knots;
            if (K == 0) continue;
            const int hg = a.kind == TAMP_MOVE_HOLD ? gslot[a.grasp] : -1;
            if (a.kind == TAMP_MOVE_HOLD)
                REQUIRE(a.grasp >= 0 && a.grasp < d.n_vars && gslot[a.grasp] >= 0, TAMP_E_INVALID, "MoveHold grasp");
            for (int j = 0; j < K; ++j) {
                REQUIRE(n_fk < TAMP_MAX_FK, TAMP_E_UNSUPPORTED, "too many robot configurations (TAMP_MAX_FK)");
                KFk& F = P.fk[n_fk++];
                F.xoff = (int16_t)(xoff[a.traj] + 7 * j);
                F.term_jl = add_term(TAMP_TERM_JL);
                F.term_cf = add_term(TAMP_TERM_CF);
                F.term_self = d.self_collision ? add_term(TAMP_TERM_SELF) : (int16_t)-1;
                F.term_kp = F.term_kr = -1;
                F.kin_inst = F.kin_grasp = -1;
                F.held_grasp = (int16_t)hg;
                F.held_obj = (int16_t)(hg >= 0 ? a.obj : -1);
                F.obb_mask = all_obb;
                F.ghost = 0;
                REQUIRE(add_partners(-1, -1, F.part_begin, F.part_count), TAMP_E_UNSUPPORTED, "too many partners");
            }
            REQUIRE(n_traj < kMaxTraj, TAMP_E_UNSUPPORTED, "too many trajectories");
            KTraj& Tj = P.traj[n_traj++];
            Tj.q1_xoff = (int16_t)xoff[a.q1]; Tj.q1_const = (int16_t)cconf[a.q1];
            Tj.q2_xoff = (int16_t)xoff[a.q2]; Tj.q2_const = (int16_t)cconf[a.q2];
            Tj.knot_xoff = (int16_t)xoff[a.traj]; Tj.n_knots = (int16_t)K;
        } else if (a.kind == TAMP_PICK || a.kind == TAMP_PLACE) {
            REQUIRE(a.obj >= 0 && a.obj < d.n_objects, TAMP_E_INVALID, "pick/place object out of range");
            REQUIRE(conf_ok(a.q1) && !d.var[a.q1].is_const, TAMP_E_UNSUPPORTED, "pick/place conf must be a free conf");
            REQUIRE(a.grasp >= 0 && a.grasp < d.n_vars && gslot[a.grasp] >= 0 && d.var[a.grasp].obj == a.obj,
                    TAMP_E_INVALID, "pick/place grasp must be a grasp variable of the object");
            REQUIRE(a.placement >= 0 && a.placement < d.n_vars && inst_of[a.placement] >= 0 &&
                    d.var[a.placement].obj == a.obj, TAMP_E_INVALID, "pick/place placement must belong to the object");
            if (a.kind == TAMP_PICK) {
                REQUIRE(held < 0, TAMP_E_INVALID, "Pick: hand not empty");
                REQUIRE(pose[a.obj] != -2, TAMP_E_INVALID, "Pick: virtual object (no initial placement)");
                REQUIRE(pose[a.obj] == inst_of[a.placement], TAMP_E_INVALID, "Pick: object is not at that placement");
            } else {
                REQUIRE(held == a.obj, TAMP_E_INVALID, "Place: object not held");
                REQUIRE(!d.var[a.placement].is_const, TAMP_E_UNSUPPORTED, "Place: placement must be free");
                REQUIRE(a.surface >= 0 && a.surface < d.n_surfaces, TAMP_E_INVALID, "Place: surface out of range");
            }
            REQUIRE(n_fk < TAMP_MAX_FK, TAMP_E_UNSUPPORTED, "too many robot configurations (TAMP_MAX_FK)");
            KFk& F = P.fk[n_fk++];
            F.xoff = (int16_t)xoff[a.q1];
            F.term_jl = add_term(TAMP_TERM_JL);
            F.term_cf = add_term(TAMP_TERM_CF);
            F.term_self = d.self_collision ? add_term(TAMP_TERM_SELF) : (int16_t)-1;
            F.term_kp = add_term(TAMP_TERM_KP);
            F.term_kr = add_term(TAMP_TERM_KR);
            F.kin_inst = (int16_t)inst_of[a.placement];
            F.kin_grasp = (int16_t)gslot[a.grasp];
            F.held_grasp = F.held_obj = -1;
            F.obb_mask = all_obb;
            F.ghost = 0;
            REQUIRE(add_partners(a.obj, -1, F.part_begin, F.part_count), TAMP_E_UNSUPPORTED, "too many partners");
            if (a.kind == TAMP_PICK) {
                held = a.obj;
                pose[a.obj] = -1;
            } else {
                const tamp_surface_desc& S = d.surface[a.surface];
                REQUIRE(n_place < kMaxPlace, TAMP_E_UNSUPPORTED, "too many Place actions");
                KPlace& Q = P.place[n_place++];
                Q.inst = (int16_t)inst_of[a.placement];
                Q.term_ss = add_term(TAMP_TERM_SS);
                Q.term_sc = add_term(TAMP_TERM_SC);
                Q.term_cp = add_term(TAMP_TERM_CP);
                Q.term_pc = -1;
                Q.surface = (int16_t)a.surface;
                Q.obb_mask = (uint16_t)(all_obb & ~(S.support_obb >= 0 ? (1u << S.support_obb) : 0u));
                REQUIRE(add_partners(a.obj, S.support_obj, Q.part_begin, Q.part_count), TAMP_E_UNSUPPORTED,
                        "too many partners");
                if (S.support_obj >= 0)
                    REQUIRE(pose[S.support_obj] >= 0 && P.inst[pose[S.support_obj]].xoff < 0, TAMP_E_UNSUPPORTED,
                            "stacking on a moved object is not supported");
                pose[a.obj] = inst_of[a.placement];
                held = -1;
            }
        } else if (a.kind == TAMP_PRESS || a.kind == TAMP_PRESS_STICK) {
            // PressButton(b, p, q) / PressButtonStick(b, o, g, p, q) (R8):
            // JL(q), CF(q) [button excluded; held stick covered by CP], [SELF], KP(q), KR(q) vs T(p) T(g),
            // SS(p) + PC(p) on the button face, and for the stick CP(p) [button excluded].
            REQUIRE(a.obj >= 0 && a.obj < d.n_objects, TAMP_E_INVALID, "press object out of range");
            REQUIRE(conf_ok(a.q1) && !d.var[a.q1].is_const, TAMP_E_UNSUPPORTED, "press conf must be a free conf");
            REQUIRE(a.grasp >= 0 && a.grasp < d.n_vars && gslot[a.grasp] >= 0 && d.var[a.grasp].obj == a.obj,
                    TAMP_E_INVALID, "press grasp must be a grasp variable of the pressing object");
            REQUIRE(a.placement >= 0 && a.placement < d.n_vars && inst_of[a.placement] >= 0 &&
                    d.var[a.placement].obj == a.obj && !d.var[a.placement].is_const, TAMP_E_INVALID,
                    "press pose must be a free placement variable of the pressing object");
            REQUIRE(a.surface >= 0 && a.surface < d.n_surfaces, TAMP_E_INVALID, "press: button face out of range");
            if (a.kind == TAMP_PRESS) {
                REQUIRE(held < 0, TAMP_E_INVALID, "PressButton: hand not empty");
                REQUIRE(pose[a.obj] == -2, TAMP_E_INVALID, "PressButton: object must be virtual (the fingertip)");
            } else {
                REQUIRE(held == a.obj, TAMP_E_INVALID, "PressButtonStick: stick not held");
            }
            const tamp_surface_desc& S = d.surface[a.surface];
            const uint16_t no_button = (uint16_t)(all_obb & ~(S.support_obb >= 0 ? (1u << S.support_obb) : 0u));
            REQUIRE(n_fk < TAMP_MAX_FK, TAMP_E_UNSUPPORTED, "too many robot configurations (TAMP_MAX_FK)");
            KFk& F = P.fk[n_fk++];
            F.xoff = (int16_t)xoff[a.q1];
            F.term_jl = add_term(TAMP_TERM_JL);
            F.term_cf = add_term(TAMP_TERM_CF);
            F.term_self = d.self_collision ? add_term(TAMP_TERM_SELF) : (int16_t)-1;
            F.term_kp = add_term(TAMP_TERM_KP);
            F.term_kr = add_term(TAMP_TERM_KR);
            F.kin_inst = (int16_t)inst_of[a.placement];
            F.kin_grasp = (int16_t)gslot[a.grasp];
            F.held_grasp = F.held_obj = -1;
            F.obb_mask = no_button;
            F.ghost = 0;
            REQUIRE(add_partners(a.obj, -1, F.part_begin, F.part_count), TAMP_E_UNSUPPORTED, "too many partners");
            REQUIRE(n_place < kMaxPlace, TAMP_E_UNSUPPORTED, "too many Place / press actions");
            KPlace& Q = P.place[n_place++];
            Q.inst = (int16_t)inst_of[a.placement];
            Q.term_ss = add_term(TAMP_TERM_SS);
            Q.term_sc = -1;
            Q.term_pc = add_term(TAMP_TERM_PC);
            Q.term_cp = a.kind == TAMP_PRESS_STICK ? add_term(TAMP_TERM_CP) : (int16_t)-1;
            Q.surface = (int16_t)a.surface;
            Q.obb_mask = no_button;
            REQUIRE(add_partners(a.obj, S.support_obj, Q.part_begin, Q.part_count), TAMP_E_UNSUPPORTED,
                    "too many partners");
        } else {
            return fail(TAMP_E_INVALID, "bad action kind");
        }
        REQUIRE(n_terms < TAMP_MAX_TERMS, TAMP_E_UNSUPPORTED, "too many hard terms (TAMP_MAX_TERMS)");
    }
    P.n_terms = n_terms;
    // Order the FK instances in pairs of identical structure (same terms, held object or not, partner count,
    // OBB mask) so that the 16-lane mapping can run the two 8-lane halves of a particle group on two FK
    // instances with warp-uniform control flow; an unmatched instance is paired with a ghost copy.
    {
        auto sig = [&](const KFk& K) {
            return std::make_tuple(K.term_cf >= 0, K.term_kp >= 0, K.term_kr >= 0, K.term_jl >= 0, K.held_grasp >= 0,
                                   K.part_count, K.obb_mask, K.term_self >= 0);
        };
        std::vector<KFk> in(P.fk, P.fk + n_fk), out;
        std::vector<bool> used(n_fk, false);
        for (int i = 0; i < n_fk; ++i) {
            if (used[i]) continue;
            used[i] = true;
            int j = -1;
            for (int k = i + 1; k < n_fk && j < 0; ++k)
                if (!used[k] && sig(in[k]) == sig(in[i])) j = k;
            out.push_back(in[i]);
            if (j >= 0) {
                used[j] = true;
                out.push_back(in[j]);
            } else {
                KFk g = in[i];
                g.ghost = 1;
                out.push_back(g);
            }
        }
        REQUIRE((int)out.size() <= TAMP_MAX_FK, TAMP_E_UNSUPPORTED, "too many robot configurations (TAMP_MAX_FK)");
        for (size_t i = 0; i < out.size(); ++i) P.fk[i] = out[i];
        n_fk = (int)out.size();
    }
    P.n_fk = n_fk;
    P.n_place = n_place;
    P.n_traj = n_traj;
    P.n_goal = d.n_goal;
    for (int k = 0; k < d.n_goal; ++k) {
        const int o = d.goal_obj[k];
        REQUIRE(o >= 0 && o < d.n_objects && pose[o] >= 0, TAMP_E_INVALID, "goal object must be placed at the end");
        P.goal_inst[k] = (int16_t)pose[o];
    }
    P.grad_scale = d.grad_scale > 0.f ? d.grad_scale : (float)(1.0 / (double)n_global);
    P.eta = d.eta;
    REQUIRE(!d.collision_smooth || d.eta > 0.f, TAMP_E_INVALID, "collision_smooth needs eta > 0");
    P.smooth = d.collision_smooth ? d.eta : 0.f;
    P.beta1 = d.beta1;
    P.beta2 = d.beta2;
    P.adam_eps = d.adam_eps;
    P.lam_goal = d.lam_goal;
    P.lam_traj = d.lam_traj;

    // sampler program (DAG order: grasps, placements, confs in declaration order; knots afterwards)
    int ns = 0;
    for (int v = 0; v < d.n_vars; ++v) {
        const tamp_var_desc& V = d.var[v];
        if (V.is_const) continue;
        KSVar& S = SP.v[ns];
        std::memset(&S, 0, sizeof(S));
        S.var_id = (int16_t)v;
        S.stream = V.rng_stream ? V.rng_stream : (uint32_t)v;
        S.xoff = (int16_t)xoff[v];
        S.slot = (int16_t)gslot[v];
        if (V.kind == TAMP_VAR_GRASP) {
            S.kind = KS_GRASP;
            S.a[0] = d.object[V.obj].grasp_xy;
            S.a[1] = d.object[V.obj].grasp_z;
            S.a[2] = d.object[V.obj].grasp_mode == 1 ? 1.f : 0.f;
            S.a[3] = d.object[V.obj].grasp_y < 0.f ? d.object[V.obj].grasp_xy : d.object[V.obj].grasp_y;
        } else if (V.kind == TAMP_VAR_PLACEMENT) {
            const tamp_surface_desc& Sf = d.surface[V.surface];
            S.kind = KS_PLACEMENT;
            S.a[0] = Sf.lo[0]; S.a[1] = Sf.lo[1]; S.a[2] = Sf.hi[0]; S.a[3] = Sf.hi[1];
            // a press pose is sampled on the whole button face (R8): contact needs only some point over it
            bool press = false;
            for (int ai = 0; ai < d.n_actions; ++ai)
                press |= (d.action[ai].kind == TAMP_PRESS || d.action[ai].kind == TAMP_PRESS_STICK) &&
                         d.action[ai].placement == v;
            S.a[4] = press ? 0.f : d.object[V.obj].footprint;
            S.a[5] = Sf.frame[0]; S.a[6] = Sf.frame[1]; S.a[7] = Sf.frame[2]; S.a[8] = Sf.frame[3];
        } else if (V.kind == TAMP_VAR_CONF) {
            S.kind = KS_CONF;
        } else {
            S.kind = KS_TRAJ;
            S.n_knots = (int16_t)V.n_knots;
            int found = -1;
            for (int ai = 0; ai < d.n_actions; ++ai)
                if ((d.action[ai].kind == TAMP_MOVE_FREE || d.action[ai].kind == TAMP_MOVE_HOLD) && d.action[ai].traj == v)
                    found = ai;
            REQUIRE(found >= 0 || V.n_knots == 0, TAMP_E_INVALID, "trajectory variable not used by a motion");
            if (found >= 0) {
                const tamp_action_desc& a = d.action[found];
                S.q1_xoff = (int16_t)xoff[a.q1]; S.q1_const = (int16_t)cconf[a.q1];
                S.q2_xoff = (int16_t)xoff[a.q2]; S.q2_const = (int16_t)cconf[a.q2];
            }
        }
        ns++;
    }
    SP.n_vars = ns;
    count_pairs(d, C);
    return check_program(C.P, C.SP);
}

// shared-memory layout of the particle kernel
static void smem_layout(tamp_ctx* c) {
    auto r4 = [](int v) { return (v + 3) & ~3; };
    const KProgram& P = c->P;
    int off = 0;
    off += r4(P.D);
    c->off_g = off;
    off += r4(P.D);
    int n_mov = 0, n_const = 0;
    bool held = false;
    for (int i = 0; i < P.n_inst; ++i) (P.inst[i].xoff >= 0 ? n_mov : n_const)++;
    for (int f = 0; f < P.n_fk; ++f) held |= P.fk[f].held_grasp >= 0;
    c->off_inst = off;                                // movable instances (kInstFloats each, 16-byte aligned)
    off += kInstFloats * n_mov;
    c->off_gT = off;                                  // grasps 3x4
    off += 12 * P.n_grasp;
    c->off_gTi = held ? off : -1;                     // inverse grasps (held objects at knots only)
    off += held ? 12 * P.n_grasp : 0;
    off = r4(off);
    c->const_floats = kInstFloats * n_const;          // constant instances: once per block
    c->fk_off = c->const_floats;                      // then the configurations' descriptors, once per block
    c->const_floats += ((P.n_fk * (int)sizeof(KFk) / 4) + 3) & ~3;
    int n_pw = 0;                                     // then the partner references' shared-memory offset words
    for (int f = 0; f < P.n_fk; ++f) n_pw = std::max(n_pw, P.fk[f].part_begin + P.fk[f].part_count);
    for (int q = 0; q < P.n_place; ++q) n_pw = std::max(n_pw, P.place[q].part_begin + P.place[q].part_count);
    c->pw_off = c->const_floats;
    c->n_pw = n_pw;
    c->const_floats += (n_pw + 3) & ~3;              // (read by the 512-bound variants: TAMP_PARTNER_TABLE)
    static_assert(sizeof(KFk) % 4 == 0, "KFk must be a whole number of floats");
    c->off_rsw = off;                                 // robot sphere centres for the SELF term (2 FK halves)
    off += P.has_self ? (c->gs == 16 ? 2 : 1) * 4 * (kGroup * TAMP_MAX_SPHERES_PER_LINK) : 0;   // per FK half
    // stride = 8 (mod 32) floats so the particles of a warp hit distinct banks on broadcasts
    int stride = ((off + 31) / 32) * 32 + 8;
    c->stride = stride;
    c->stride_bytes = stride * (int)sizeof(float);
}

static size_t mv_bytes(const tamp_ctx* c) { return (size_t)((c->n + 31) & ~(int64_t)31) * c->P.D * 4; }

static void ws_layout(tamp_ctx* c) {
    const int64_t n = c->n;
    const int D = c->P.D, G = c->P.n_grasp;
    c->n_keys = n > 65536 ? n : 65536;
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o = align256(o + bytes); return r; };
    c->o_x = take((size_t)n * D * 4);
    // Adam moments: padded to whole 32-particle tiles (the serial mapping's layout, mv_w32_index)
    c->o_m = take(mv_bytes(c));
    c->o_v = take(mv_bytes(c));
    c->o_grasp = take((size_t)n * G * 12 * 4);
    c->o_inv = take((size_t)n);
    c->o_cls = take((size_t)n);
    c->o_cost = take((size_t)n * 4);
    c->o_ka = take((size_t)c->n_keys * 8);
    c->o_kb = take((size_t)c->n_keys * 8);
    c->o_pa = take((size_t)c->n_keys * 4);
    c->o_pb = take((size_t)c->n_keys * 4);
    c->o_coords = take((size_t)3 * (D > 0 ? D : 1) * 4);
    c->o_counts = take((size_t)(TAMP_MAX_TERMS + 2) * 4);
    c->o_stage = take((size_t)1024 * (D + 4) * 4);
    // IK restarts: per Kin conf, the list of particles whose first IK run did not converge (+ its length)
    int n_kin = 0;
    if (c->ik_iters > 0 && c->ik_seeds > 1)
        for (int f = 0; f < c->P.n_fk; ++f)
            if ((c->P.fk[f].term_kp >= 0 || c->P.fk[f].term_kr >= 0) && !c->P.fk[f].ghost) ++n_kin;
    c->o_iklist = take((size_t)2 * n_kin * n * 4);                 // ping-pong lists of the restart rounds
    c->o_ikn = take((size_t)(n_kin > 0 ? n_kin : 1) * 8 * 4);      // list lengths, <= 7 rounds + 1
    c->o_ikbest = take((size_t)n_kin * n * 4);                     // best restart score so far
    c->total = o;
}

static bool is_host_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeUnregistered;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

static KArgs base_args(tamp_ctx* c) {
    KArgs A;
    std::memset(&A, 0, sizeof(A));
    A.x = c->at<float>(c->o_x);
    A.m = c->at<float>(c->o_m);
    A.v = c->at<float>(c->o_v);
    A.grasp = c->at<float>(c->o_grasp);
    A.invalid = c->at<uint8_t>(c->o_inv);
    const float* coords = c->at<float>(c->o_coords);
    A.lr = coords;
    A.lo = coords + c->P.D;
    A.hi = coords + 2 * c->P.D;
    A.n = c->n;
    A.gofs = c->gofs;
    A.stride = c->stride;
    A.off_g = c->off_g;
    A.off_inst = c->off_inst;
    A.const_floats = c->const_floats;
    A.fk_off = c->fk_off;
    A.pw_off = c->pw_off;
    A.n_pw = c->n_pw;
    A.off_gT = c->off_gT;
    A.off_gTi = c->off_gTi;
    A.off_rsw = c->off_rsw;
    A.bsync = c->gs == 1 ? c->bsync : 0;
    A.smem_floats = (int32_t)(c->smem / sizeof(float));
    return A;
}

// ------------------------------------------------------------------------------------------------
// C ABI
// ------------------------------------------------------------------------------------------------
extern "C" {

int32_t tamp_abi_version(void) { return TAMP_ABI_VERSION; }

const char* tamp_last_error(void) { return g_err.c_str(); }

size_t tamp_sizeof_desc(void) { return sizeof(tamp_problem_desc); }

size_t tamp_sizeof_info(void) { return sizeof(tamp_info); }

uint64_t tamp_kernel_launches(void) { return tamp::launch_count(); }

tamp_status tamp_query_workspace(const tamp_problem_desc* desc, int64_t n_local, size_t* bytes) {
    if (!desc || !bytes) return fail(TAMP_E_INVALID, "null argument");
    if (n_local < 1 || n_local > (1ll << 30)) return fail(TAMP_E_INVALID, "n_local must be in [1, 2^30]");
    tamp_ctx tmp;
    Compiled C;
    tamp_status s = compile(*desc, n_local, C);
    if (s != TAMP_OK) return s;
    tmp.P = C.P;
    tmp.n = n_local;
    tmp.ik_iters = desc->ik_iters;
    tmp.ik_seeds = desc->ik_seeds ? desc->ik_seeds : 1;
    ws_layout(&tmp);
    *bytes = tmp.total;
    return TAMP_OK;
}

tamp_status tamp_init_problem(const tamp_problem_desc* desc, int device, int64_t n_local, int64_t global_offset,
                              int64_t n_global, void* d_workspace, size_t ws_bytes, tamp_ctx** out) {
    if (!desc || !out) return fail(TAMP_E_INVALID, "null argument");
    *out = nullptr;
    if (n_local < 1 || n_local > (1ll << 30)) return fail(TAMP_E_INVALID, "n_local must be in [1, 2^30]");
    if (global_offset < 0 || n_global < global_offset + n_local || n_global > (1ll << 30))
        return fail(TAMP_E_INVALID, "need 0 <= global_offset, global_offset + n_local <= n_global <= 2^30");
    if (!d_workspace || (reinterpret_cast<uintptr_t>(d_workspace) & 255))
        return fail(TAMP_E_INVALID, "workspace must be a 256-byte aligned device pointer");
    Compiled C;
    tamp_status s = compile(*desc, n_global, C);
    if (s != TAMP_OK) return s;
    tamp_ctx* c = new tamp_ctx();
    c->device = device;
    c->n = n_local;
    c->gofs = global_offset;
    c->nglob = n_global;
    c->P = C.P;
    c->SP = C.SP;
    std::memcpy(c->term_kind, C.term_kind, sizeof(c->term_kind));
    std::memcpy(c->term_action, C.term_action, sizeof(c->term_action));
    c->pairs_sb = C.pairs_sb;
    c->pairs_ss = C.pairs_ss;
    c->n_robot_spheres = desc->robot.n_spheres;
    if (desc->ik_iters < 0 || desc->ik_iters > 1000 || !(desc->ik_damping >= 0.f)) {
        delete c;
        return fail(TAMP_E_INVALID, "ik_iters must be in [0, 1000] and ik_damping >= 0");
    }
    c->ik_iters = desc->ik_iters;
    c->ik_damping = desc->ik_damping;
    c->ik_seeds = desc->ik_seeds ? desc->ik_seeds : 1;
    if (c->ik_seeds != 1 && c->ik_seeds != 2 && c->ik_seeds != 4 && c->ik_seeds != 8) {
        delete c;
        return fail(TAMP_E_INVALID, "ik_seeds must be 0, 1, 2, 4 or 8");
    }
    if (desc->lanes_per_particle != 0 && desc->lanes_per_particle != 1 && desc->lanes_per_particle != 4 &&
        desc->lanes_per_particle != 8 && desc->lanes_per_particle != 16) {
        delete c;
        return fail(TAMP_E_INVALID, "lanes_per_particle must be 0, 1, 4, 8 or 16");
    }
    // auto: 8 lanes (one per link frame) -- measured faster than 16 on every config, even at 8K particles
    // (profiles/r1: the 16-lane mapping doubles the FK/kin instruction count for little latency gain)
    {
        int n_fk_real = 0;
        for (int f = 0; f < c->P.n_fk; ++f) n_fk_real += !c->P.fk[f].ghost;
        // 16 lanes (two FK instances at a time) pays off for knot-heavy skeletons (config 4: 48 FK
        // instances); 4 lanes (two link frames per lane, 8 particles per warp) for launches that take many
        // waves when a 512-thread block (128 particles) fits shared memory (config 1 at 1M: +10 %);
        // 8 lanes elsewhere (sweeps 9, 13)
        c->gs = desc->lanes_per_particle ? desc->lanes_per_particle : (n_fk_real >= 24 ? 16 : 8);
        // serial mapping (one thread per particle) for many particles of a small skeleton: no redundant
        // per-particle work; config 1 at 64K-1M particles +27-34 % over the lane mappings (profiles/README.md),
        // but 4x slower on the collision-heavy Tetris skeletons (D = 72), so only for small D
        if (!desc->lanes_per_particle && n_local >= 65536 && c->P.D <= 32 && !c->P.has_self) {
            bool held = false;
            for (int f = 0; f < c->P.n_fk; ++f) held |= c->P.fk[f].held_grasp >= 0;
            if (!held) c->gs = 1;
        }
    }
    ws_layout(c);
    smem_layout(c);
    if (!desc->lanes_per_particle && c->gs == 8) {
        int n_sm = 148, smem_optin = 227 * 1024;
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, device);
        cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
        cudaGetLastError();
        const bool many_waves = n_local > (int64_t)n_sm * 4 * (768 / 8);
        // (small skeletons only: on the Tetris skeletons the 4-lane blocks were 1.6x slower than 8 lanes in
        // 896-thread blocks, profiles/r2_sweep_cfg5_262k.txt)
        if (many_waves && c->P.D <= 32 && 128 * c->stride_bytes + 4 * c->const_floats + 4096 <= smem_optin) c->gs = 4;
    }
    if (c->gs == 1) {
        // serial mapping (particle_serial.cuh): one thread per particle, per-thread state in shared memory
        bool held = false;
        for (int f = 0; f < c->P.n_fk; ++f) held |= c->P.fk[f].held_grasp >= 0;
        int smem_optin = 227 * 1024;
        cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
        cudaGetLastError();
        c->threads = desc->block_threads ? desc->block_threads : 128;
        const int maxt = (TAMP_SERIAL_PP && c->P.smooth <= 0.f && serial_program_pp(c->P)) ? kSerialThreadsPP : kSerialThreads;
        if (c->threads % 32 || c->threads < 32 || c->threads > maxt) {
            delete c;
            return fail(TAMP_E_INVALID, "block_threads must be a multiple of 32 in [32, 512] for 1 lane per particle "
                                        "(pick-place class programs: [32, 640])");
        }
        // block-synchronous configurations (default): one large block per SM whose warps walk the ~100 KB kernel
        // body together and share the instruction cache (`no_instruction` was the top stall with independent
        // small blocks: 1.6 cycles per issued instruction, profiles/README.md)
        c->bsync = desc->block_sync >= 0 ? (desc->block_sync ? 1 : 0) : 1;
        // auto: with barriers, the largest block that fits one per SM (shared memory holds the per-particle
        // state, columns of pitch threads + 1); without, the block size with the most resident warps per SM
        if (!desc->block_threads) {
            int smem_sm = 228 * 1024;
            cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
            cudaGetLastError();
            const int regs = std::max(32, serial_kernel_regs(TAMP_SERIAL_PP && c->P.smooth <= 0.f && serial_program_pp(c->P)));
            int n_sm = 148;
            cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, device);
            cudaGetLastError();
            int best_w = -1;
            double best_cost = 1e300;
            for (int t = 32; t <= (c->bsync ? maxt : 128); t += 32) {
                const size_t sb = serial_smem_bytes(c->P, t, true) + 4096;   // + static smem, reserved
                if (sb > (size_t)smem_optin) continue;
                const int by_smem = (int)((size_t)smem_sm / sb);
                const int by_regs = 65536 / (((regs + 7) & ~7) * t);
                const int blocks = c->bsync ? std::min(std::min(by_smem, by_regs), 1) : std::min(std::min(by_smem, by_regs), 32);
                if (blocks < 1) continue;
                const int w = blocks * (t / 32);
                if (c->bsync) {
                    // balanced waves (as for the lane mappings): W waves of w resident warps per SM cost W (w + 20)
                    // -- the per-SM rate w / (w + 20) fitted to the serial kernel's warp sweep (9 / 11 / 13 / 15
                    // warps: 2268 / 2729 / 2869 / 3117 particles per ms per wave)
                    const int64_t nb = (n_local + t - 1) / t;
                    const int64_t waves = (nb + n_sm - 1) / n_sm;
                    const double cost = (double)waves * (w + 20);
                    if (cost < best_cost || (cost == best_cost && t > c->threads)) { best_cost = cost; c->threads = t; }
                } else if (w > best_w || (w == best_w && t > c->threads)) {
                    best_w = w;
                    c->threads = t;
                }
            }
        }
        c->smem = serial_smem_bytes(c->P, c->threads, true);
        if (c->P.has_self || held || c->smem + 4096 > (size_t)smem_optin) {
            delete c;
            return fail(TAMP_E_UNSUPPORTED, "1 lane per particle: no SELF term, no held objects at knots, and the "
                                            "per-particle state must fit shared memory");
        }
    } else {
        // launch configuration of the particle kernel.  Auto: block-synchronous phases with one large block
        // per SM holding that SM's share of the particles (all warps of an SM walk the same code region ->
        // shared instruction cache), bounded by 768 threads and by shared memory.
        int n_sm = 148, smem_optin = 227 * 1024;
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, device);
        cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
        cudaGetLastError();
        const int ppw = 32 / c->gs;                                     // particles per warp
        const int static_smem = 4096 + 4 * c->const_floats;   // + block-shared constant instances
        // __launch_bounds__ of the variants: 8 lanes up to 1024 threads (hinge; 768 for the smooth cost), else 512
        const int max_threads = C.P.smooth > 0.f ? (c->gs == 8 ? 768 : 512) : (c->gs == 8 ? 1024 : (c->gs == 16 ? 768 : 512));
        int max_pp = std::min(max_threads / c->gs, (smem_optin - static_smem) / c->stride_bytes);
        max_pp = (max_pp / ppw) * ppw;
        if (desc->block_threads) {
            if (desc->block_threads % 32 || desc->block_threads < 32 || desc->block_threads > max_threads) {
                delete c;
                return fail(TAMP_E_INVALID, "block_threads must be a multiple of 32 in [32, 1024] for 8 lanes, 768 for 16 "
                                            "lanes (768 / 512 with the smooth cost), 512 for 4 lanes");
            }
            c->threads = desc->block_threads;
        } else {
            // measured (profiles/README.md, sweeps 8-10):
            //  - if every particle of the launch is resident at once with one block per SM holding that SM's
            //    share, that block with phase-level barriers is best (config 2 at 8K);
            //  - otherwise the block size with the lowest estimated launch time over balanced waves (below).
            int64_t pp = (n_local + n_sm - 1) / n_sm;                      // this SM's share
            pp = ((pp + ppw - 1) / ppw) * ppw;
            c->bsync = 1;
            if (pp <= max_pp) {
                c->threads = (int)std::min<int64_t>(std::max<int64_t>(pp, 4 * ppw), std::max(max_pp, ppw)) * c->gs;
            } else {
                auto blocks_per_sm = [&](int t) {
                    const int regs = std::max(32, particle_kernel_regs(c->gs, t));   // variant run by t threads
                    const int ppb = t / c->gs;
                    const int by_regs = 65536 / (((regs + 7) & ~7) * t);
                    const int by_smem = (smem_optin + 1024) / (ppb * c->stride_bytes + static_smem + 1024);
                    return std::min(std::min(by_regs, by_smem), 32);
                };
                // multi-wave: the block size whose launch is estimated fastest.  Each wave is balanced (the block
                // shrunk so every wave is equally full) and costs W x (w + 20) for W waves of w resident warps per
                // SM: the rate per SM grows as w / (w + 20), fitted to config 3 (76 particles per SM = 19 warps,
                // 3 waves: 2.29 ms; 96 = 24 warps, 3 waves: 2.59 ms).  Fewer, fuller waves win: config 3 at
                // 32,768 runs 2 waves of 111 particles (888 threads, the 896-bound variant) instead of 3 of 74.
                // (ties go to the larger block: fewer, larger blocks per SM share the instruction cache -- 4
                // independent 128-thread blocks ran config 4 at half the speed of one 448-thread block)
                double best_cost = 1e300;
                int best_t = 128, best_b = 1, best_W = 1;
                for (int t = (max_threads / 32) * 32; t >= 128; t -= 32) {
                    const int ppb = t / c->gs;
                    if (ppb % ppw || ppb > max_pp) continue;
                    const int bps = blocks_per_sm(t);
                    if (bps < 1) continue;
                    const int64_t cap = (int64_t)n_sm * bps * ppb;              // particles per wave
                    const int64_t W = (n_local + cap - 1) / cap;
                    const int64_t p_sm = (n_local + (int64_t)n_sm * W - 1) / ((int64_t)n_sm * W);
                    const double w = (double)p_sm * c->gs / 32.0;
                    const double cost = (double)W * (w + 20.0);
                    if (cost < best_cost - 1e-9) { best_cost = cost; best_t = t; best_b = bps; best_W = (int)W; }
                }
                int64_t ppb = (n_local + (int64_t)n_sm * best_W * best_b - 1) / ((int64_t)n_sm * best_W * best_b);
                ppb = ((ppb + ppw - 1) / ppw) * ppw;
                c->threads = (int)std::min<int64_t>(ppb * c->gs, best_t);
            }
        }
        if (c->threads / c->gs > max_pp) {
            delete c;
            return fail(TAMP_E_UNSUPPORTED, "block too large for shared memory");
        }
        if (desc->block_sync > 2) {
            delete c;
            return fail(TAMP_E_INVALID, "block_sync must be -1 (auto) or 0..2");
        }
        if (desc->block_threads && desc->block_sync < 0) c->bsync = 2;
        if (desc->block_sync >= 0) c->bsync = desc->block_sync;
        c->smem = (size_t)(c->threads / c->gs) * c->stride_bytes + 4 * (size_t)c->const_floats;
    }
    if (ws_bytes < c->total) {
        delete c;
        return fail(TAMP_E_NOMEM, "workspace too small: need " + std::to_string(c->total) + " bytes");
    }

    c->base = static_cast<char*>(d_workspace);
    c->ws_bytes = ws_bytes;
    c->coords.reserve(3 * C.lr.size());
    c->coords.insert(c->coords.end(), C.lr.begin(), C.lr.end());
    c->coords.insert(c->coords.end(), C.lo.begin(), C.lo.end());
    c->coords.insert(c->coords.end(), C.hi.begin(), C.hi.end());
    DeviceGuard g(device);
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, d_workspace) != cudaSuccess || a.type != cudaMemoryTypeDevice) {
        cudaGetLastError();
        delete c;
        return fail(TAMP_E_INVALID, "workspace is not device memory");
    }
    *out = c;
    return TAMP_OK;
}

tamp_status tamp_get_info(const tamp_ctx* c, tamp_info* out) {
    if (!c || !out) return fail(TAMP_E_INVALID, "null argument");
    std::memset(out, 0, sizeof(*out));
    out->D = c->P.D;
    out->n_hard = c->P.n_terms;
    out->n_grasp = c->P.n_grasp;
    out->n_fk = c->P.n_fk;
    for (int i = 0; i < c->P.n_terms; ++i) {
        out->term_kind[i] = c->term_kind[i];
        out->term_action[i] = c->term_action[i];
    }
    out->n_local = c->n;
    out->global_offset = c->gofs;
    out->n_global = c->nglob;
    out->t = c->t;
    out->pairs_sphere_obb = c->pairs_sb;
    out->pairs_sphere_sphere = c->pairs_ss;
    int n_kin = 0, n_seg = 0;
    int n_fk_real = 0;
    for (int f = 0; f < c->P.n_fk; ++f) {
        n_kin += c->P.fk[f].term_kp >= 0 && !c->P.fk[f].ghost;
        n_fk_real += !c->P.fk[f].ghost;
    }
    out->n_fk = n_fk_real;
    for (int i = 0; i < c->P.n_traj; ++i) n_seg += c->P.traj[i].n_knots + 1;
    out->n_kin = n_kin;
    out->n_place = c->P.n_place;
    out->n_goal_pairs = c->P.n_goal * (c->P.n_goal - 1) / 2;
    out->n_traj_seg = n_seg;
    out->n_robot_spheres = c->n_robot_spheres;
    out->lanes_per_particle = c->gs;
    out->block_threads = c->threads;
    out->block_sync = c->bsync;
    {
        int64_t per_conf = 0, n_self = 0;
        for (int i = 0; i < kGroup * TAMP_MAX_SPHERES_PER_LINK; ++i) per_conf += __builtin_popcount(c->P.self_mask[i]);
        for (int f = 0; f < c->P.n_fk; ++f) n_self += c->P.fk[f].term_self >= 0 && !c->P.fk[f].ghost;
        out->pairs_self = per_conf / 2 * n_self;
    }
    return TAMP_OK;
}

// the per-coordinate lr | lo | hi arrays: copied into the workspace on the stream of the first call that may precede
// every other (sample / set_state), so that init has no hidden synchronisation (tamp.h conventions)
static cudaError_t upload_coords(tamp_ctx* c, cudaStream_t st) {
    if (c->coords_on_device || c->coords.empty()) return cudaSuccess;
    cudaError_t e = cudaMemcpyAsync(c->at<float>(c->o_coords), c->coords.data(), c->coords.size() * 4,
                                    cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) c->coords_on_device = true;
    return e;
}

tamp_status tamp_sample_particles(tamp_ctx* c, uint64_t seed, void* stream) {
    if (!c) return fail(TAMP_E_INVALID, "null context");
    DeviceGuard g(c->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    CUDA_TRY(upload_coords(c, st), "sample: upload bounds");
    CUDA_TRY(launch_sample(c->SP, c->at<float>(c->o_x), c->at<float>(c->o_grasp), c->n, c->gofs, seed, st), "sample");
    CUDA_TRY(launch_ik(c->P, c->SP, c->at<float>(c->o_x), c->at<float>(c->o_grasp), c->n, c->gofs, seed, c->ik_iters,
                       c->ik_damping, c->ik_seeds, c->at<int32_t>(c->o_iklist), c->at<int32_t>(c->o_ikn),
                       c->at<float>(c->o_ikbest), st),
             "sample: IK");
    CUDA_TRY(cudaMemsetAsync(c->base + c->o_m, 0, mv_bytes(c), st), "sample: zero m");
    CUDA_TRY(cudaMemsetAsync(c->base + c->o_v, 0, mv_bytes(c), st), "sample: zero v");
    CUDA_TRY(cudaMemsetAsync(c->base + c->o_inv, 0, (size_t)c->n, st), "sample: zero invalid");
    c->t = 0;
    c->ready = true;
    c->checked = false;
    return TAMP_OK;
}

// n_steps fused Adam steps in launches of <= kMaxStepsPerLaunch; with check_last, the last launch also runs the
// Eq. 3 check of the final state (lane mappings) into the context's class / cost / counts buffers
static tamp_status run_optimize(tamp_ctx* c, int32_t n_steps, cudaStream_t st, bool check_last) {
    KArgs A = base_args(c);
    if (check_last) {
        A.out_cls = c->at<uint8_t>(c->o_cls);
        A.out_cost = c->at<float>(c->o_cost);
        A.out_counts = c->at<int32_t>(c->o_counts);
        CUDA_TRY(cudaMemsetAsync(A.out_counts, 0, (TAMP_MAX_TERMS + 2) * 4, st), "optimize+check: zero counts");
    }
    for (int32_t done = 0; done < n_steps;) {
        const int32_t k = std::min<int32_t>(n_steps - done, kMaxStepsPerLaunch);
        A.n_steps = k;
        A.t0 = c->t;
        A.check_after = check_last && done + k == n_steps ? 1 : 0;
        for (int i = 0; i < k; ++i) {   // Adam bias corrections (Kingma & Ba): 1 / (1 - beta^t), t = t0 + i + 1
            const double t = (double)(c->t + i + 1);
            A.rbc1[i] = (float)(1.0 / (1.0 - std::pow((double)c->P.beta1, t)));
            A.rbc2[i] = (float)(1.0 / (1.0 - std::pow((double)c->P.beta2, t)));
        }
        CUDA_TRY(launch_particle(MODE_OPT, c->gs, c->bsync, c->threads, c->P, A, c->smem, st), "optimize");
        c->t += k;
        c->checked = A.check_after != 0;
        done += k;
    }
    return TAMP_OK;
}

tamp_status tamp_optimize_step(tamp_ctx* c, int32_t n_steps, void* stream) {
    if (!c) return fail(TAMP_E_INVALID, "null context");
    if (!c->ready) return fail(TAMP_E_STATE, "optimize before sample/set_state");
    if (n_steps < 0) return fail(TAMP_E_INVALID, "n_steps must be >= 0");
    if (n_steps == 0) return TAMP_OK;
    DeviceGuard g(c->device);
    return run_optimize(c, n_steps, static_cast<cudaStream_t>(stream), false);
}

static tamp_status run_check(tamp_ctx* c, cudaStream_t st) {
    KArgs A = base_args(c);
    A.out_cls = c->at<uint8_t>(c->o_cls);
    A.out_cost = c->at<float>(c->o_cost);
    A.out_counts = c->at<int32_t>(c->o_counts);
    CUDA_TRY(cudaMemsetAsync(A.out_counts, 0, (TAMP_MAX_TERMS + 2) * 4, st), "check: zero counts");
    CUDA_TRY(launch_particle(MODE_CHECK, c->gs, c->bsync, c->threads, c->P, A, c->smem, st), "check");
    c->checked = true;
    return TAMP_OK;
}

tamp_status tamp_check_satisfied(tamp_ctx* c, uint8_t* cls, int32_t* counts, void* stream) {
    if (!c) return fail(TAMP_E_INVALID, "null context");
    if (!c->ready) return fail(TAMP_E_STATE, "check before sample/set_state");
    if (!counts) return fail(TAMP_E_INVALID, "counts must not be NULL");
    DeviceGuard g(c->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    tamp_status s = run_check(c, st);
    if (s != TAMP_OK) return s;
    const size_t nb = (size_t)(c->P.n_terms + 2) * 4;
    CUDA_TRY(cudaMemcpyAsync(counts, c->at<int32_t>(c->o_counts), nb, cudaMemcpyDefault, st), "check: counts copy");
    if (cls) CUDA_TRY(cudaMemcpyAsync(cls, c->at<uint8_t>(c->o_cls), (size_t)c->n, cudaMemcpyDefault, st), "check: cls copy");
    if (is_host_ptr(counts) || is_host_ptr(cls)) CUDA_TRY(cudaStreamSynchronize(st), "check: sync");
    return TAMP_OK;
}

tamp_status tamp_optimize_and_check(tamp_ctx* c, int32_t n_steps, uint8_t* cls, int32_t* counts, void* stream) {
    if (!c) return fail(TAMP_E_INVALID, "null context");
    if (!c->ready) return fail(TAMP_E_STATE, "optimize before sample/set_state");
    if (n_steps < 1) return fail(TAMP_E_INVALID, "n_steps must be >= 1");
    if (!counts) return fail(TAMP_E_INVALID, "counts must not be NULL");
    DeviceGuard g(c->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    {
        tamp_status s = run_optimize(c, n_steps, st, true);
        if (s != TAMP_OK) return s;
    }
    const size_t nb = (size_t)(c->P.n_terms + 2) * 4;
    CUDA_TRY(cudaMemcpyAsync(counts, c->at<int32_t>(c->o_counts), nb, cudaMemcpyDefault, st), "check: counts copy");
    if (cls) CUDA_TRY(cudaMemcpyAsync(cls, c->at<uint8_t>(c->o_cls), (size_t)c->n, cudaMemcpyDefault, st), "check: cls copy");
    if (is_host_ptr(counts) || is_host_ptr(cls)) CUDA_TRY(cudaStreamSynchronize(st), "check: sync");
    return TAMP_OK;
}

tamp_status tamp_best_k(tamp_ctx* c, int32_t k, float* records, void* stream) {
    if (!c) return fail(TAMP_E_INVALID, "null context");
    if (!c->ready) return fail(TAMP_E_STATE, "best_k before sample/set_state");
    if (!records || k < 1 || k > 1024 || k > c->n) return fail(TAMP_E_INVALID, "need 1 <= k <= min(1024, n_local)");
    DeviceGuard g(c->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (!c->checked) {       // classes and costs of the current state (a check since the last step reuses them)
        tamp_status s = run_check(c, st);
        if (s != TAMP_OK) return s;
    }
    unsigned long long *ka = c->at<unsigned long long>(c->o_ka), *kb = c->at<unsigned long long>(c->o_kb);
    int32_t *pa = c->at<int32_t>(c->o_pa), *pb = c->at<int32_t>(c->o_pb);
    CUDA_TRY(launch_make_keys(c->at<uint8_t>(c->o_cls), c->at<float>(c->o_cost), c->n, c->gofs, ka, pa, st), "best_k: keys");
    unsigned long long* kr;
    int32_t* pr;
    CUDA_TRY(launch_topk(ka, pa, kb, pb, c->n, k, st, &kr, &pr), "best_k: sort");
    float* stage = c->at<float>(c->o_stage);
    CUDA_TRY(launch_gather_particles(pr, kr, k, c->at<float>(c->o_x), c->at<float>(c->o_cost), c->P.D, c->gofs, stage, st),
             "best_k: gather");
    CUDA_TRY(cudaMemcpyAsync(records, stage, (size_t)k * (c->P.D + 4) * 4, cudaMemcpyDefault, st), "best_k: copy");
    if (is_host_ptr(records)) CUDA_TRY(cudaStreamSynchronize(st), "best_k: sync");
    return TAMP_OK;
}

tamp_status tamp_merge_best_k(tamp_ctx* c, const float* d_in, int32_t n_in, int32_t k, float* d_out, void* stream) {
    if (!c || !d_in || !d_out) return fail(TAMP_E_INVALID, "null argument");
    if (n_in < 1 || n_in > 65536 || k < 1 || k > n_in || k > 1024) return fail(TAMP_E_INVALID, "need 1 <= k <= n_in <= 65536, k <= 1024");
    DeviceGuard g(c->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int width = c->P.D + 4;
    unsigned long long *ka = c->at<unsigned long long>(c->o_ka), *kb = c->at<unsigned long long>(c->o_kb);
    int32_t *pa = c->at<int32_t>(c->o_pa), *pb = c->at<int32_t>(c->o_pb);
    CUDA_TRY(launch_record_keys(d_in, n_in, width, ka, pa, st), "merge: keys");
    unsigned long long* kr;
    int32_t* pr;
    CUDA_TRY(launch_topk(ka, pa, kb, pb, n_in, k, st, &kr, &pr), "merge: sort");
    CUDA_TRY(launch_gather_records(pr, k, d_in, width, d_out, st), "merge: gather");
    return TAMP_OK;
}

static size_t merge_scratch_layout(int32_t n_in, size_t* o_kb, size_t* o_pa, size_t* o_pb) {
    const size_t n = (size_t)n_in;
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o = align256(o + bytes); return r; };
    take(n * 8);                      // keys a at offset 0
    *o_kb = take(n * 8);
    *o_pa = take(n * 4);
    *o_pb = take(n * 4);
    return o;
}

tamp_status tamp_merge_scratch_bytes(int32_t n_in, size_t* bytes) {
    if (!bytes || n_in < 1 || n_in > 65536) return fail(TAMP_E_INVALID, "need bytes and 1 <= n_in <= 65536");
    size_t a, b, c;
    *bytes = merge_scratch_layout(n_in, &a, &b, &c);
    return TAMP_OK;
}

tamp_status tamp_merge_records(const float* d_in, int32_t n_in, int32_t k, int32_t D, float* d_out, void* d_scratch,
                               size_t scratch_bytes, void* stream) {
    if (!d_in || !d_out || !d_scratch) return fail(TAMP_E_INVALID, "null argument");
    if (n_in < 1 || n_in > 65536 || k < 1 || k > n_in || k > 1024) return fail(TAMP_E_INVALID, "need 1 <= k <= n_in <= 65536, k <= 1024");
    if (D < 0 || D > TAMP_MAX_D) return fail(TAMP_E_INVALID, "D out of range");
    if (reinterpret_cast<uintptr_t>(d_scratch) & 255) return fail(TAMP_E_INVALID, "scratch must be 256-byte aligned");
    size_t o_kb, o_pa, o_pb;
    if (scratch_bytes < merge_scratch_layout(n_in, &o_kb, &o_pa, &o_pb)) return fail(TAMP_E_NOMEM, "merge scratch too small");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    char* base = static_cast<char*>(d_scratch);
    unsigned long long *ka = reinterpret_cast<unsigned long long*>(base), *kb = reinterpret_cast<unsigned long long*>(base + o_kb);
    int32_t *pa = reinterpret_cast<int32_t*>(base + o_pa), *pb = reinterpret_cast<int32_t*>(base + o_pb);
    const int width = D + 4;
    CUDA_TRY(launch_record_keys(d_in, n_in, width, ka, pa, st), "merge: keys");
    unsigned long long* kr;
    int32_t* pr;
    CUDA_TRY(launch_topk(ka, pa, kb, pb, n_in, k, st, &kr, &pr), "merge: sort");
    CUDA_TRY(launch_gather_records(pr, k, d_in, width, d_out, st), "merge: gather");
    return TAMP_OK;
}

tamp_status tamp_eval(tamp_ctx* c, float* J, float* soft, float* Jc, float* grad, void* stream) {
    if (!c) return fail(TAMP_E_INVALID, "null context");
    if (!c->ready) return fail(TAMP_E_STATE, "eval before sample/set_state");
    for (const void* p : {(const void*)J, (const void*)soft, (const void*)Jc, (const void*)grad})
        if (p && is_host_ptr(p)) return fail(TAMP_E_INVALID, "tamp_eval outputs must be device pointers");
    DeviceGuard g(c->device);
    KArgs A = base_args(c);
    A.out_J = J;
    A.out_soft = soft;
    A.out_Jc = Jc;
    A.out_grad = grad;
    CUDA_TRY(launch_particle(MODE_EVAL, c->gs, c->bsync, c->threads, c->P, A, c->smem, static_cast<cudaStream_t>(stream)), "eval");
    return TAMP_OK;
}

// Adam moments between the caller's [n][D] layout and the context's: [n][D] for the lane mappings, 32-particle tiles
// for the serial mapping (mv_w32_index) -- converted by a kernel for device-accessible buffers, on the host (through
// a staging copy, synchronous) for host buffers
static cudaError_t get_moments(tamp_ctx* c, float* dst, size_t off, cudaStream_t st) {
    const size_t nd = (size_t)c->n * c->P.D * 4;
    if (c->gs != 1) return cudaMemcpyAsync(dst, c->base + off, nd, cudaMemcpyDefault, st);
    if (!is_host_ptr(dst)) return launch_mv_layout(c->at<float>(off), dst, c->n, c->P.D, 0, st);
    std::vector<float> t(mv_bytes(c) / 4);
    cudaError_t e = cudaMemcpyAsync(t.data(), c->base + off, mv_bytes(c), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    const int D = c->P.D;
    for (int64_t p = 0; p < c->n; ++p)
        for (int d = 0; d < D; ++d) dst[p * D + d] = t[mv_w32_index(p, d, D)];
    return cudaSuccess;
}
static cudaError_t set_moments(tamp_ctx* c, const float* src, size_t off, cudaStream_t st) {
    const size_t nd = (size_t)c->n * c->P.D * 4;
    if (c->gs != 1) return cudaMemcpyAsync(c->base + off, src, nd, cudaMemcpyDefault, st);
    if (!is_host_ptr(src)) return launch_mv_layout(src, c->at<float>(off), c->n, c->P.D, 1, st);
    const int D = c->P.D;
    std::vector<float> t(mv_bytes(c) / 4, 0.f);
    for (int64_t p = 0; p < c->n; ++p)
        for (int d = 0; d < D; ++d) t[mv_w32_index(p, d, D)] = src[p * D + d];
    cudaError_t e = cudaMemcpyAsync(c->base + off, t.data(), mv_bytes(c), cudaMemcpyHostToDevice, st);
    return e == cudaSuccess ? cudaStreamSynchronize(st) : e;   // the staging vector must outlive the copy
}

tamp_status tamp_get_state(tamp_ctx* c, float* x, float* m, float* v, float* grasp, uint8_t* invalid, int32_t* t,
                           void* stream) {
    if (!c) return fail(TAMP_E_INVALID, "null context");
    if (!c->ready) return fail(TAMP_E_STATE, "get_state before sample/set_state");
    DeviceGuard g(c->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t nd = (size_t)c->n * c->P.D * 4;
    bool host = false;
    if (x) { CUDA_TRY(cudaMemcpyAsync(x, c->base + c->o_x, nd, cudaMemcpyDefault, st), "get x"); host |= is_host_ptr(x); }
    if (m) { CUDA_TRY(get_moments(c, m, c->o_m, st), "get m"); host |= is_host_ptr(m); }
    if (v) { CUDA_TRY(get_moments(c, v, c->o_v, st), "get v"); host |= is_host_ptr(v); }
    if (grasp && c->P.n_grasp) {
        CUDA_TRY(cudaMemcpyAsync(grasp, c->base + c->o_grasp, (size_t)c->n * c->P.n_grasp * 48, cudaMemcpyDefault, st), "get grasp");
        host |= is_host_ptr(grasp);
    }
    if (invalid) {
        CUDA_TRY(cudaMemcpyAsync(invalid, c->base + c->o_inv, (size_t)c->n, cudaMemcpyDefault, st), "get invalid");
        host |= is_host_ptr(invalid);
    }
    if (t) *t = c->t;
    if (host) CUDA_TRY(cudaStreamSynchronize(st), "get_state: sync");
    return TAMP_OK;
}

tamp_status tamp_set_state(tamp_ctx* c, const float* x, const float* m, const float* v, const float* grasp,
                           const uint8_t* invalid, int32_t t, void* stream) {
    if (!c) return fail(TAMP_E_INVALID, "null context");
    if (!x) return fail(TAMP_E_INVALID, "set_state needs x");
    if (t < 0) return fail(TAMP_E_INVALID, "t must be >= 0");
    if (!grasp && c->P.n_grasp && !c->ready) return fail(TAMP_E_STATE, "first set_state must provide grasps");
    DeviceGuard g(c->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    CUDA_TRY(upload_coords(c, st), "set_state: upload bounds");
    const size_t nd = (size_t)c->n * c->P.D * 4;
    CUDA_TRY(cudaMemcpyAsync(c->base + c->o_x, x, nd, cudaMemcpyDefault, st), "set x");
    if (m) CUDA_TRY(set_moments(c, m, c->o_m, st), "set m");
    else CUDA_TRY(cudaMemsetAsync(c->base + c->o_m, 0, mv_bytes(c), st), "zero m");
    if (v) CUDA_TRY(set_moments(c, v, c->o_v, st), "set v");
    else CUDA_TRY(cudaMemsetAsync(c->base + c->o_v, 0, mv_bytes(c), st), "zero v");
    if (grasp && c->P.n_grasp)
        CUDA_TRY(cudaMemcpyAsync(c->base + c->o_grasp, grasp, (size_t)c->n * c->P.n_grasp * 48, cudaMemcpyDefault, st), "set grasp");
    if (invalid) CUDA_TRY(cudaMemcpyAsync(c->base + c->o_inv, invalid, (size_t)c->n, cudaMemcpyDefault, st), "set invalid");
    else CUDA_TRY(cudaMemsetAsync(c->base + c->o_inv, 0, (size_t)c->n, st), "zero invalid");
    if (is_host_ptr(x) || is_host_ptr(m) || is_host_ptr(v) || is_host_ptr(grasp) || is_host_ptr(invalid))
        CUDA_TRY(cudaStreamSynchronize(st), "set_state: sync");
    c->t = t;
    c->ready = true;
    c->checked = false;
    return TAMP_OK;
}

double tamp_plan_heuristic(const int32_t* counts, int32_t n_hard, double penalty) {
    if (!counts || n_hard <= 0) return 0.0;
    double h = 0.0;
    for (int32_t c = 0; c < n_hard; ++c) h += counts[c] > 0 ? (double)counts[c] : penalty;
    return h / n_hard;
}

void tamp_destroy(tamp_ctx* c) { delete c; }

}  // extern "C"
