// tamp_program.h -- compiled form of a skeleton's CSP, as read by the sm_100a kernels.
//
// Built once on the host by tamp_init_problem (tamp_api.cu) from tamp_problem_desc; passed to
// every kernel launch by value as a __grid_constant__ parameter (uniform data served by the
// constant cache).  Per-coordinate arrays (lr, lo, hi) live in the device workspace.
// Internal to libtamp: not part of the C ABI.
#pragma once
#include <stdint.h>
#include "../../include/tamp.h"

namespace tamp {

constexpr int kMaxInst = 24;          // object instances: (object, pose source) pairs
constexpr int kMaxPlace = 16;         // Place actions
constexpr int kMaxTraj = 32;          // motions carrying knots
constexpr int kMaxPartners = 1024;    // collision partner instance references
constexpr int kMaxConstConf = 8;      // constant confs referenced by trajectories (q0)
constexpr int kGroup = 8;             // lanes per particle: one per link frame (7 joints + tool)
// Adam moments of the serial mapping (one thread per particle): 32-particle tiles, coordinate-major inside a tile
// (element (p, d) at ((p / 32) * D + d) * 32 + p % 32; the arrays hold ceil(n / 32) * 32 * D floats).  The lane
// mappings use [n][D]; tamp_get_state / tamp_set_state convert.
__host__ __device__ inline int64_t mv_w32_index(int64_t p, int d, int D) {
    return ((p >> 5) * D + d) * 32 + (p & 31);
}
constexpr int kMaxStepsPerLaunch = 64; // fused Adam steps per particle-kernel launch
constexpr int kInstFloats = 56;        // shared memory per object instance: pose 3x4, bounding sphere, 8 spheres, wrench

// One robot configuration evaluated per particle-step: a Pick/Place conf or a trajectory knot.
struct KFk {
    int16_t xoff;                     // offset of the 7 joint values in x
    int16_t term_jl, term_cf;         // hard-term ids (-1 none)
    int16_t term_kp, term_kr;
    int16_t kin_inst;                 // Kin target placement instance (-1 none)
    int16_t kin_grasp;                // grasp slot of the Kin target
    int16_t held_grasp;               // grasp slot of the object held at this knot (-1 none)
    int16_t held_obj;                 // object id of the held object
    int16_t part_begin, part_count;   // collision partner instances: partners[part_begin ...]
    uint16_t obb_mask;                // OBBs checked against the robot (and held object)
    int16_t ghost;                    // 1 = padding copy of its pair partner (results discarded)
    int16_t term_self;                // robot self-collision term (-1 none)
};

// An object at a pose: constant (xoff < 0, pose[]) or a placement variable at x[xoff .. xoff+4).
struct KInst {
    int16_t obj;
    int16_t xoff;
    int16_t slot;                     // index among the movable (xoff >= 0, per particle) or the constant (per block)
                                      // instances: the kernel keeps kInstFloats floats of shared memory for each
    float pose[4];                    // x y z yaw (constant instances)
};

// StablePlace + CFreePlace of one Place action, or ValidPress / ValidStickPress (+ CFreePlace of the held
// stick) of one PressButton / PressButtonStick action: SS always, SC (Place) or PC (press), CP unless -1.
struct KPlace {
    int16_t inst;                     // instance of the placed / pressing object at its placement variable
    int16_t term_ss, term_sc, term_cp, term_pc;
    int16_t surface;
    int16_t part_begin, part_count;
    uint16_t obb_mask;                // OBBs checked (support excluded)
};

// TrajLength(q1, k_1..k_K, q2) of one motion.  Endpoint xoff < 0 -> constant conf (index const_idx).
struct KTraj {
    int16_t q1_xoff, q1_const, q2_xoff, q2_const;
    int16_t knot_xoff, n_knots;
};

struct KSurface { float frame[4]; float lo[2], hi[2]; float cy, sy; };   // cy, sy: cos / sin of the frame yaw
struct KObb {                          // oriented box: world pose R (row-major), centre c, half extents h
    float R[9];
    float c[3];
    float h[3];
    float rad;                         // |h|: bounding-sphere radius
    int32_t aligned;                   // R is exactly the identity (axis-aligned fast path)
    float lo[3], hi[3];                // aligned boxes: corners c -/+ h grown by kCornerSlack (conservative reject test)
};
constexpr double kCornerSlack = 2e-5;  // m: >> the fp32 rounding of w - c - h at |coordinates| <= kMaxCoord
constexpr double kMaxCoord = 100.0;

struct KProgram {
    int32_t D, n_terms, n_fk, n_inst, n_place, n_traj, n_goal, n_grasp, n_obb;
    float grad_scale, eta, beta1, beta2, adam_eps, lam_goal, lam_traj;
    float smooth;                        // CHOMP-smooth collision cost width (= eta) or 0 = hinge
    KFk fk[TAMP_MAX_FK];
    KInst inst[kMaxInst];
    KPlace place[kMaxPlace];
    KTraj traj[kMaxTraj];
    int16_t partners[kMaxPartners];
    int16_t goal_inst[TAMP_MAX_GOAL];
    float term_lam[TAMP_MAX_TERMS];
    float term_eps[TAMP_MAX_TERMS];
    KSurface surf[TAMP_MAX_SURFACES];
    KObb obb[TAMP_MAX_OBB];
    float const_conf[kMaxConstConf][7];
    // robot: per lane l of a particle group, the fixed transform F_{l+1} (3x4 row-major; base folded
    // into F_1) or, for lane 7, the tool transform F_ee; and the spheres attached to that frame.
    float F[kGroup][12];
    float Finv[kGroup][12];              // F^-1 of each (serial mapping: backward sweep over the links)
    // modified-DH numbers of joints 2..7 (index 1..6): (a_{j-1}, d_j, cos alpha_{j-1}, sin alpha_{j-1}), F[j] =
    // Rx(alpha) Tx(a) Tz(d) -- the serial mapping composes / inverts these factors directly (dh_fwd / dh_bwd);
    // index 0 is unused (F[0] also carries the base)
    float dh[TAMP_NJ][4];
    float rsph[kGroup][TAMP_MAX_SPHERES_PER_LINK][4];
    int32_t rsph_n[kGroup];
    float jlo[TAMP_NJ], jhi[TAMP_NJ];
    // objects
    float osph[TAMP_MAX_OBJECTS][TAMP_MAX_OBJ_SPHERES][4];
    int32_t osph_n[TAMP_MAX_OBJECTS];
    float obound[TAMP_MAX_OBJECTS][4];   // bounding sphere of each object's spheres (object frame xyz, radius)
    // self-collision: bit t of self_mask[s] = check robot spheres s, t (packed ids: link lane * 4 + k)
    uint32_t self_mask[kGroup * TAMP_MAX_SPHERES_PER_LINK];
    float lbound[kGroup][4];             // bounding sphere of each link frame's spheres (link frame xyz, radius)
    int32_t has_self;
};

// Particle-initialisation program (K1).
enum { KS_GRASP = 0, KS_PLACEMENT = 1, KS_CONF = 2, KS_TRAJ = 3 };
struct KSVar {
    uint32_t stream;                            // Philox counter word 2 (rng_stream or the variable index)
    int16_t kind, var_id, xoff, slot;          // slot: grasp slot for KS_GRASP
    int16_t q1_xoff, q1_const, q2_xoff, q2_const, n_knots;
    float a[12];                                // sampler parameters (see k_sample)
};
struct KSampleProgram {
    int32_t n_vars, D, n_grasp;
    float jlo[TAMP_NJ], jhi[TAMP_NJ];
    float const_conf[kMaxConstConf][7];
    KSVar v[TAMP_MAX_VARS];
};

// Workspace carve-up (byte offsets from the caller's base pointer; 256-B aligned).
struct Workspace {
    size_t x, m, v, grasp, invalid, cls, cost, keys_a, keys_b, coords, counts, stage, total;
    int64_t n_pad;
    int32_t stage_bytes;
};

// Arguments of the particle kernel (K2/K3/eval).
enum { MODE_OPT = 0, MODE_EVAL = 1, MODE_CHECK = 2 };

struct KArgs {
    float* x;              // [n][D]
    float* m;              // [n][D]
    float* v;              // [n][D]
    const float* grasp;    // [n][G][12]
    uint8_t* invalid;      // [n]
    const float* lr;       // [D]
    const float* lo;       // [D]
    const float* hi;       // [D]
    int64_t n;
    int64_t gofs;
    int32_t stride, off_g, off_inst, off_gT, off_gTi, off_rsw;   // per-particle shared memory (floats); off_gTi < 0:
                                                               // no held object at a knot, no inverse grasps
    int32_t const_floats;  // block-shared constant instances at the start of dynamic shared memory, then the
    int32_t fk_off;        // configurations' descriptors (KFk[n_fk], lane mappings) at float offset fk_off
    int32_t pw_off, n_pw;  // and the partner references' offset words (int[n_pw], TAMP_PARTNER_TABLE)
    int32_t n_steps, t0;
    int32_t bsync;         // serial mapping: block barriers per configuration / phase (shared i-cache)
    int32_t check_after;   // MODE_OPT: run the Eq. 3 check of the final state in the same launch
    int32_t smem_floats;   // dynamic shared memory of the launch (device-check builds verify every carve-out)
    // reciprocal Adam bias corrections 1 / (1 - beta^t) for the (<= kMaxStepsPerLaunch) steps of this launch,
    // computed on the host in double precision
    float rbc1[64], rbc2[64];
    // MODE_EVAL outputs (nullable)
    float* out_J;
    float* out_soft;
    float* out_Jc;
    float* out_grad;
    // MODE_CHECK outputs
    uint8_t* out_cls;
    float* out_cost;
    int32_t* out_counts;
};

}  // namespace tamp
