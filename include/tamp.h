/*
 * tamp.h -- C ABI of the B200-native cuTAMP particle-optimisation hot path (libtamp.so).
 *
 * What the calls compute (PAPER.md = /root/reference/PAPER.md, "P:n" = line n):
 *   A plan skeleton pi induces a continuous CSP whose free parameters (placements, arm
 *   configurations, trajectory knots; grasps are sampled and frozen) form a
 *   particle x.  Each particle's cost is the penalty relaxation
 *       J(x) = sum_c lambda_c J_c(x) + sum_c' lambda_c' c'(x)                   (Eq. 2)
 *   a particle satisfies the CSP iff  AND_c J_c(x) <= eps_c                      (Eq. 3)
 *   and a batch is optimised on the mean cost with Adam                          (Eq. 4)
 *   after compositional sampling initialises it.
 *   Readings where the paper is silent follow SURVEY.md §8(c) L1-L25 / DESIGN.md.
 *
 * Conventions (all calls):
 *   - Every call returns tamp_status; none aborts or exits.  tamp_last_error() gives a
 *     thread-local message for the last non-OK status.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Calls are
 *     stream-ordered and asynchronous unless a HOST buffer is passed (see below); asynchronous
 *     device faults surface on a later call as TAMP_E_CUDA.
 *   - Buffer arguments marked "device or host" may be device pointers or host pointers
 *     (pageable or pinned).  With host pointers the library stages through its workspace and
 *     the call synchronises `stream` before returning.
 *   - Ownership: the caller owns the device workspace and all buffers.  The library owns only
 *     the opaque host-side context.  A context is bound to one device; it is not thread-safe.
 *   - Call order: init -> sample (or set_state) -> {optimize | check | best_k | eval | get/set}*.
 *     Anything else returns TAMP_E_STATE.
 *   - Layouts: particle state is particle-major, x[i][d] at x[i*D + d] (row i = particle i, the
 *     stacked variable matrices X_i of P:483-484 side by side).  Grasps: grasp[i][k][12] = the
 *     3x4 row-major transform T(g_k) of particle i in its object's frame.
 */
#ifndef TAMP_H_
#define TAMP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TAMP_ABI_VERSION 4

/* compiled limits of the sm_100a kernels (exceeding one returns TAMP_E_UNSUPPORTED) */
#define TAMP_NJ 7                     /* 7-DOF arm */
#define TAMP_MAX_ROBOT_SPHERES 32     /* 8 links x 4 spheres: one link per lane of an 8-lane group */
#define TAMP_MAX_SPHERES_PER_LINK 4
#define TAMP_MAX_OBB 16
#define TAMP_MAX_OBJECTS 8
#define TAMP_MAX_OBJ_SPHERES 8
#define TAMP_MAX_SURFACES 8
#define TAMP_MAX_VARS 96
#define TAMP_MAX_ACTIONS 64
#define TAMP_MAX_GOAL 8
#define TAMP_MAX_D 384                /* optimised floats per particle */
#define TAMP_MAX_TERMS 256            /* hard constraint terms */
#define TAMP_MAX_FK 64                /* robot configurations evaluated per particle (confs + knots) */
#define TAMP_MAX_GRASPS 8
#define TAMP_MAX_KNOTS 8

typedef enum {
    TAMP_OK = 0,
    TAMP_E_INVALID = 1,      /* bad argument or descriptor (message says which) */
    TAMP_E_CUDA = 2,         /* CUDA runtime error (message has cudaGetErrorString) */
    TAMP_E_NOMEM = 3,        /* workspace too small */
    TAMP_E_STATE = 4,        /* call-order violation */
    TAMP_E_UNSUPPORTED = 5   /* descriptor exceeds a compiled limit */
} tamp_status;

/* variable kinds */
enum { TAMP_VAR_CONF = 0, TAMP_VAR_PLACEMENT = 1, TAMP_VAR_GRASP = 2, TAMP_VAR_TRAJ = 3 };
/* actions of Listing 1 and of the Stick Button domain:
   PressButton(b, p, q): hand empty; `obj` = the robot's virtual fingertip object (an object with no
     constant initial placement: never in the scene), `grasp` = its grasp variable (TCP pose in the
     fingertip frame), `placement` = the press pose p (a placement variable of the fingertip object),
     `surface` = the button's top face (support_obb = the button); conf q1.
   PressButtonStick(b, o, g, p, q): stick o held with grasp g; `placement` = the stick's pose p while
     pressing (a placement variable of o), `surface` = the button's top face; conf q1.  o stays held. */
enum { TAMP_MOVE_FREE = 0, TAMP_PICK = 1, TAMP_MOVE_HOLD = 2, TAMP_PLACE = 3, TAMP_PRESS = 4,
       TAMP_PRESS_STICK = 5 };
/* hard-constraint term kinds (SURVEY §8(c) term table):
   JL joint limits (Motion); CF robot collision (CFreeTraj/CFreeHold/CFreeTrajHold,
   P:1029-1031); KP/KR kinematics position/rotation (Kin); SS/SC stable-place support /
   containment; CP CFreePlace; SELF robot self-collision ("does not cause
   robot self-collisions", tolerance 0 P:1132; enabled by desc.self_collision);
   PC press contact (ValidPress / ValidStickPress, R8): min over the pressing
   object's spheres of dist_from_bounds(xy in the button-face frame, lo, hi); with SS (the object's bottom
   at the face height) it says "some point of the fingertip / stick touches the button's top face". */
enum { TAMP_TERM_JL = 0, TAMP_TERM_CF = 1, TAMP_TERM_KP = 2, TAMP_TERM_KR = 3,
       TAMP_TERM_SS = 4, TAMP_TERM_SC = 5, TAMP_TERM_CP = 6, TAMP_TERM_SELF = 7, TAMP_TERM_PC = 8,
       TAMP_N_TERM_KINDS = 9 };

/* Serial 7-DOF arm, modified (Craig) DH: frame_j = frame_{j-1} Rx(alpha_{j-1}) Tx(a_{j-1}) Tz(d_j) Rz(q_j);
   tool/TCP = frame_7 Tz(flange_d) Rz(tcp_yaw) Tz(tcp_d); frame_0 = Trans(base xyz) Rz(base yaw).
   Spheres: centre in the frame of link sphere_link[s] (1..7 = link frames, 8 = tool frame),
   radius > 0; at most TAMP_MAX_SPHERES_PER_LINK per link. */
typedef struct {
    float dh[TAMP_NJ][3];                 /* (a_{j-1}, d_j, alpha_{j-1}) */
    float flange_d, tcp_yaw, tcp_d;
    float base[4];                        /* x y z yaw */
    float joint_lo[TAMP_NJ], joint_hi[TAMP_NJ];
    int32_t n_spheres;
    float sphere[TAMP_MAX_ROBOT_SPHERES][4];
    int32_t sphere_link[TAMP_MAX_ROBOT_SPHERES];
    uint32_t self_mask[TAMP_MAX_ROBOT_SPHERES];   /* bit j of self_mask[i]: sphere pair (i, j) is checked by
                                                     the SELF term (symmetric; typically non-adjacent links) */
} tamp_robot_desc;

/* static oriented box ("oriented bounding boxes"): centre, half extents > 0 and its orientation:
   rot = the box-to-world rotation (3x3, row-major; must be orthonormal with det +1 to 1e-4, else TAMP_E_INVALID),
   or all nine entries 0: the rotation Rz(yaw) about the world z axis.  |center_k| + half_k <= 100 m
   (TAMP_E_UNSUPPORTED beyond: the kernels' conservative reject test is sized for fp32 rounding at that scale) */
typedef struct { float center[3]; float yaw; float half[3]; float rot[9]; } tamp_obb_desc;

/* movable object as spheres in its frame (origin = bottom centre, L15); sampler parameters:
   footprint = radius shrinking placement regions; top-down grasp TCP at (u*grasp_xy, v*grasp_y, grasp_z),
   u, v uniform in [-1, 1] (grasp_y < 0: grasp_y = grasp_xy);
   grasp_mode 0 = top-down 4-DOF, 1 = 6-DOF (top or one of the 4 sides, approach through the vertical axis
   at height grasp_z; "top-down 4-DOF or 6-DOF poses").  An object with no constant initial
   placement variable is virtual (the fingertip of PressButton): never in the scene, never a collision
   partner. */
typedef struct {
    int32_t n_spheres;
    float sphere[TAMP_MAX_OBJ_SPHERES][4];
    float footprint, grasp_xy, grasp_z;
    int32_t grasp_mode;
    float grasp_y;
} tamp_object_desc;

/* placement surface: frame (x, y, z_top, yaw) in the world, rectangle lo/hi in that frame;
   support_obb / support_obj (-1 none) are excluded from CFreePlace (L3) */
typedef struct {
    float frame[4];
    float lo[2], hi[2];
    int32_t support_obb, support_obj;
} tamp_surface_desc;

/* continuous skeleton parameter.  is_const marks the bold constants q0 / p0:
   value = conf (7) or placement (x y z yaw).  placement: obj, surface (sampler), clamp lo/hi (x y z yaw,
   +-INFINITY allowed).  grasp: obj.  traj: n_knots free knots (<= TAMP_MAX_KNOTS). */
typedef struct {
    int32_t kind, is_const, obj, surface, n_knots;
    float value[7];
    float lo[4], hi[4];
    uint32_t rng_stream;                  /* sampler stream (Philox counter word 2): 0 = the variable's index;
                                             equal streams + equal sampler inputs give equal samples, which is
                                             how a planner reuses a shared subgraph's samples */
} tamp_var_desc;

/* ground action (Listing 1); unused fields = -1.  Pick/Place/Press use q1 as their conf;
   MoveFree/MoveHold go q1 -> q2 through traj (-1 = deferred motion). */
typedef struct { int32_t kind, obj, grasp, placement, surface, q1, q2, traj; } tamp_action_desc;

typedef struct {
    int32_t abi_version;                  /* = TAMP_ABI_VERSION */
    tamp_robot_desc robot;
    int32_t n_obb;
    tamp_obb_desc obb[TAMP_MAX_OBB];
    int32_t n_objects;
    tamp_object_desc object[TAMP_MAX_OBJECTS];
    int32_t n_surfaces;
    tamp_surface_desc surface[TAMP_MAX_SURFACES];
    int32_t n_vars;
    tamp_var_desc var[TAMP_MAX_VARS];
    int32_t n_actions;
    tamp_action_desc action[TAMP_MAX_ACTIONS];
    int32_t n_goal;                       /* MinimizeObjDist goal objects; 0 = none */
    int32_t goal_obj[TAMP_MAX_GOAL];
    float lam[TAMP_N_TERM_KINDS];         /* lambda_c > 0 */
    float eps[TAMP_N_TERM_KINDS];         /* eps_c >= 0 */
    float lam_goal, lam_traj;             /* soft-cost weights (L7, L8) */
    float eta;                            /* collision activation distance >= 0 (L1) */
    float beta1, beta2, adam_eps;         /* Adam (L9) */
    float lr_conf, lr_pos, lr_yaw, lr_knot;
    float grad_scale;                     /* <= 0: use 1 / n_global (Eq. 4) */
    int32_t lanes_per_particle;           /* kernel mapping (schedule only; results agree to fp32 rounding):
                                             1 = one thread per particle (serial mapping, no SELF / held objects),
                                             4 / 8 = lanes per configuration's link frames, 16 = two
                                             configurations at a time; 0 = auto */
    int32_t block_threads;                /* particle-kernel block size (multiple of 32, <= 768; <= 512 for 4 / 16
                                             lanes, <= 128 for 1); 0 = auto */
    int32_t block_sync;                   /* block barriers of the link mappings: 0 none, 1 one per step after
                                             the configuration loop, 2 + after every configuration; -1 auto (1) */
    int32_t self_collision;               /* 1: add a SELF term after every CF term */
    int32_t collision_smooth;             /* 1: CHOMP-smooth collision cost instead of the hinge:
                                             p - eta/2 (p > eta), p^2/(2 eta) (0 < p <= eta), p = r + eta - sd;
                                             needs eta > 0 */
    int32_t ik_iters;                     /* conditional IK sampler: damped-least-squares iterations
                                             per Pick/Place/Press conf inside tamp_sample_particles; 0 = uniform confs */
    float ik_damping;                     /* DLS damping mu (dq = J^T (J J^T + mu^2 I)^-1 e) */
    int32_t ik_seeds;                     /* IK restarts per conf, 1, 2, 4 or 8 (0 = 1), solved in parallel (cuRobo's
                                             solver is multi-seed): seed 0 starts from the uniform conf sample,
                                             seed s >= 1 from a fresh uniform conf (Philox blocks 2s, 2s+1 of the conf's
                                             stream); kept: the first seed whose final position / rotation error is
                                             <= 1e-3 m / 1e-3 rad, else the one with the smallest sum of the two
                                             (lowest seed on ties) -- DESIGN.md R6 */
} tamp_problem_desc;

/* what the compiled CSP looks like (term order = DESIGN.md "canonical term order") */
typedef struct {
    int32_t D;                            /* optimised floats per particle */
    int32_t n_hard;                       /* hard terms (length of Jc rows, counts = n_hard + 2) */
    int32_t n_grasp;                      /* frozen grasps per particle */
    int32_t n_fk;                         /* arm configurations evaluated per particle-step */
    int32_t term_kind[TAMP_MAX_TERMS];    /* TAMP_TERM_* of each hard term */
    int64_t n_local, global_offset, n_global;
    int32_t t;                            /* Adam step counter */
    /* work per particle-step: collision pairs evaluated, Kin residual
       pairs, Place actions, obj_dist pairs, TrajLength segments */
    int64_t pairs_sphere_obb, pairs_sphere_sphere;
    int32_t n_kin, n_place, n_goal_pairs, n_traj_seg, n_robot_spheres;
    int32_t lanes_per_particle;           /* mapping chosen for the particle kernel */
    int32_t block_threads, block_sync;    /* launch configuration chosen for the particle kernel */
    int64_t pairs_self;                   /* robot self-collision sphere pairs per particle-step */
    int32_t term_action[TAMP_MAX_TERMS];  /* index of the skeleton action that emitted each hard term */
} tamp_info;

typedef struct tamp_ctx tamp_ctx;

int32_t tamp_abi_version(void);
const char* tamp_last_error(void);
/* sizeof(tamp_problem_desc) / sizeof(tamp_info) as compiled into the library (binding self-check) */
size_t tamp_sizeof_desc(void);
size_t tamp_sizeof_info(void);
/* number of kernels this process has launched through libtamp (evidence for bench's gpu_launches) */
uint64_t tamp_kernel_launches(void);

/* Device workspace bytes needed for n_local particles of this problem. */
tamp_status tamp_query_workspace(const tamp_problem_desc* desc, int64_t n_local, size_t* bytes);

/* Compile the skeleton (host) and bind a context to `device` and the caller-owned
   workspace (>= tamp_query_workspace bytes, 256-B aligned).  This rank owns global particles
   [global_offset, global_offset + n_local) of n_global.  The descriptor is copied.  No device work
   and no synchronisation: the per-coordinate bounds are copied into the workspace on the stream of the first
   tamp_sample_particles / tamp_set_state. */
tamp_status tamp_init_problem(const tamp_problem_desc* desc, int device, int64_t n_local,
                              int64_t global_offset, int64_t n_global,
                              void* d_workspace, size_t ws_bytes, tamp_ctx** out);
tamp_status tamp_get_info(const tamp_ctx* ctx, tamp_info* out);

/* InitializeParticles (Alg. 1): Philox4x32-10 counter RNG (key = seed, counter =
   (global index lo, hi, variable stream = rng_stream or the variable index, block)); grasps top-down and frozen, placements uniform on the
   surface region, confs uniform within joint limits, then (ik_iters > 0) the conditional IK sampler
    toward each Pick/Place/Press conf's Kin target, knots linear interpolation.  Resets Adam
   (m = v = 0, t = 0) and the invalid flags. */
tamp_status tamp_sample_particles(tamp_ctx* ctx, uint64_t seed, void* stream);

/* OptimizeParticles (Alg. 1): n_steps fused Adam steps on Eq. 4 (gradient scale
   grad_scale), each followed by projection to the variable bounds (L11).  A particle whose cost
   or gradient becomes non-finite is marked invalid (sticky) and no longer updated. */
tamp_status tamp_optimize_step(tamp_ctx* ctx, int32_t n_steps, void* stream);

/* IsGoalSatisfied (Eq. 3) at the current x: cls[i] = 0 satisfying, 1 not, 2 invalid;
   counts[c] = #particles with J_c <= eps_c for each hard term c (the n_satisfying of Eq. 5),
   counts[n_hard] = #satisfying, counts[n_hard + 1] = #invalid.  cls may be NULL.
   cls [n_local] u8 and counts [n_hard + 2] i32: device or host. */
tamp_status tamp_check_satisfied(tamp_ctx* ctx, uint8_t* cls, int32_t* counts, void* stream);

/* tamp_optimize_step(n_steps) followed by tamp_check_satisfied, as one call (Alg. 1's optimise-then-check
   interval): identical results; the check of the final state runs inside the last optimisation
   launch (no second launch re-loading the state).  n_steps >= 1; cls may be NULL;
   buffers as for tamp_check_satisfied. */
tamp_status tamp_optimize_and_check(tamp_ctx* ctx, int32_t n_steps, uint8_t* cls, int32_t* counts, void* stream);

/* Best k particles of this rank (GetSatisfyingParticles) at the current x, sorted by
   key (class, cost, global index) ascending, cost = soft plan cost if satisfying else J.
   records [k][D + 4] floats (device or host): [class, cost, global_idx_lo, global_idx_hi
   (int32 bit patterns), x[0..D)].  k <= n_local, k <= 1024. */
tamp_status tamp_best_k(tamp_ctx* ctx, int32_t k, float* records, void* stream);

/* Deterministic global top-k of n_in records (e.g. all-gathered from G ranks) with the same key, using
   ctx's workspace as scratch (D = ctx's D).  d_in [n_in][D + 4], d_out [k][D + 4]: device pointers.
   k <= n_in <= 65536, k <= 1024. */
tamp_status tamp_merge_best_k(tamp_ctx* ctx, const float* d_in, int32_t n_in, int32_t k, float* d_out,
                              void* stream);

/* The same merge without a context (SURVEY §8(b)'s stateless form): records of width D + 4, caller-owned device
   scratch of >= tamp_merge_scratch_bytes(n_in) bytes (256-B aligned), on the current device.  Same results as
   tamp_merge_best_k.  Errors: TAMP_E_INVALID (arguments), TAMP_E_NOMEM (scratch too small). */
tamp_status tamp_merge_scratch_bytes(int32_t n_in, size_t* bytes);
tamp_status tamp_merge_records(const float* d_in, int32_t n_in, int32_t k, int32_t D, float* d_out, void* d_scratch,
                               size_t scratch_bytes, void* stream);

/* Test / inspection (not on the timed path): per-particle J, soft cost, Jc [n_local][n_hard] and
   the UNSCALED gradient dJ/dx [n_local][D] at the current x.  Any output may be NULL.  Device only. */
tamp_status tamp_eval(tamp_ctx* ctx, float* J, float* soft, float* Jc, float* grad, void* stream);

/* State access (checkpoint / parity).  x, m, v [n_local][D]; grasp [n_local][n_grasp][12];
   invalid [n_local] u8.  Device or host; any pointer may be NULL (get: skipped; set: m, v, invalid
   NULL -> zero, grasp NULL -> keep, x must be given).  set_state also sets the Adam counter t.
   The context's internal layout of m and v is its own (the 1-lane-per-particle mapping keeps them in 32-particle
   tiles); these calls always exchange [n_local][D] and convert (a kernel for device buffers; for host buffers a
   host reorder through a staging copy, synchronous). */
tamp_status tamp_get_state(tamp_ctx* ctx, float* x, float* m, float* v, float* grasp,
                           uint8_t* invalid, int32_t* t, void* stream);
tamp_status tamp_set_state(tamp_ctx* ctx, const float* x, const float* m, const float* v,
                           const float* grasp, const uint8_t* invalid, int32_t t, void* stream);

/* Plan-feasibility heuristic (Eq. 5) from the satisfied counts of tamp_check_satisfied (host
   pointer, all-reduced over ranks): H = (1/n_hard) sum_c h_c, h_c = counts[c] if counts[c] > 0 else
   penalty (Lambda_penalty, "a large negative penalty").  n_hard = 0 -> 0. */
double tamp_plan_heuristic(const int32_t* counts, int32_t n_hard, double penalty);

void tamp_destroy(tamp_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* TAMP_H_ */
