/*
 * kamino_b200.h — C-ABI of the B200-native per-step PADMM forward-dynamics solve.
 *
 * This is the drop-in boundary for the reference's C++ solver/world/step API
 * (/root/reference/proj/include/loopdyn/ *.hpp).  Every entry point below names
 * the reference interface it replaces (file:line).  Signatures carry only plain
 * pointers, sizes and POD structs — no torch, no Eigen, no C++ types — so the
 * reference-side C++ wrapper (include/loopdyn_b200/) or a ctypes
 * binding can call it directly.
 *
 * Conventions (reference se3.hpp:14-18): quaternions are Hamilton, serialized
 * scalar-first [w,x,y,z]; a pose maps body to world; twists are world-frame
 * [linear; angular].  Batch storage is the reference WorldBatch layout
 * (batch.hpp:41-42): 7 doubles per body pose [x y z qw qx qy qz], 6 doubles per
 * body twist, per-world prefix-sum offsets in world order.
 *
 * Errors: every function returns an int status (KD_OK = 0).  The reference
 * throws ModelError{Code} (model.hpp:76-94), SceneError (scene.hpp:74-77) and
 * std::runtime_error on an LLT failure (delassus.cpp:209-215); here those are
 * status codes plus a thread-local message from kd_last_error().  Solver
 * non-convergence and CR breakdown are flags in kd_step_diag, never errors
 * (padmm.cpp:154-157, delassus.cpp:196).
 */
#ifndef KAMINO_B200_H
#define KAMINO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes --------------------------------------------------------- */
enum {
  KD_OK = 0,
  /* ModelError::Code (model.hpp:78-88), offset by 1 so 0 stays "ok" */
  KD_ERR_MODEL_INVALID_REFERENCE = 1,
  KD_ERR_MODEL_NON_UNIT_AXIS = 2,
  KD_ERR_MODEL_BAD_INERTIA = 3,
  KD_ERR_MODEL_BAD_LIMITS = 4,
  KD_ERR_MODEL_UNSUPPORTED_ON_JOINT_TYPE = 5,
  KD_ERR_MODEL_BAD_GEOMETRY = 6,
  KD_ERR_MODEL_UNSUPPORTED_COLLISION_PAIR = 7,
  KD_ERR_MODEL_WRONG_JOINT_TYPE = 8,
  KD_ERR_MODEL_DUPLICATE_NAME = 9,
  /* runtime */
  KD_ERR_INVALID_ARGUMENT = 20,
  KD_ERR_CUDA = 21,
  KD_ERR_SPD_FAILURE = 22, /* "Delassus factorization failed on an SPD system" (delassus.cpp:212) */
  KD_ERR_CAPACITY = 23,
  KD_ERR_NO_DEVICE = 24
};

/* ---- scene description (mirrors SceneDescription, scene.hpp:15-72) --------- */
typedef struct kd_body_desc {
  const char* name;
  double mass;
  double inertia[9];          /* row-major 3x3 body-frame inertia about the COM */
  double position[3];
  double orientation[4];      /* [w,x,y,z] */
  double linear_velocity[3];
  double angular_velocity[3];
} kd_body_desc;

typedef struct kd_joint_desc {
  const char* name;
  const char* type;           /* "fixed" | "revolute" | "prismatic" | "spherical" */
  const char* parent;         /* body name or "world" */
  const char* child;
  double parent_position[3];
  double parent_orientation[4];
  double child_position[3];
  double child_orientation[4];
  double axis[3];
  int32_t has_limits;
  double lower, upper;
  double kp, kd;
  int32_t has_target;         /* std::optional<double> target (scene.hpp:34) */
  double target;
  double target_rate;
  double armature;
  double damping;
} kd_joint_desc;

typedef struct kd_geom_desc {
  const char* body;           /* "world" for planes */
  const char* shape;          /* "sphere" | "plane" | "box" */
  double radius;
  double half_extents[3];
  double normal[3];
  double offset;
  double mu;
  double restitution;
} kd_geom_desc;

typedef struct kd_scene_desc {
  const char* name;
  double gravity[3];
  int32_t n_bodies;
  const kd_body_desc* bodies;
  int32_t n_joints;
  const kd_joint_desc* joints;
  int32_t n_geoms;
  const kd_geom_desc* geoms;
} kd_scene_desc;

/* ---- step configuration (StepConfig stepper.hpp:16-34 + PadmmConfig padmm.hpp:8-17) */
enum { KD_INTEGRATOR_SEMI_IMPLICIT_EULER = 0, KD_INTEGRATOR_MOREAU_JEAN = 1 };
enum { KD_BACKEND_DENSE = 0, KD_BACKEND_MATRIX_FREE = 1, KD_BACKEND_AUTO = 2 }; /* delassus.hpp:85 */
#define KD_DENSE_ROW_CROSSOVER 300 /* kDenseRowCrossover, delassus.hpp:89 */

typedef struct kd_step_config {
  double dt;                      /* 1/240 */
  int32_t integrator;             /* KD_INTEGRATOR_* (default semi-implicit Euler) */
  int32_t backend;                /* KD_BACKEND_* (default Auto) */
  double eta;                     /* 1e-6 */
  double rho;                     /* 0.1 (padmm.hpp:10) */
  double eps;                     /* 1e-6 */
  int32_t max_iters;              /* 200 */
  int32_t acceleration;           /* 1 */
  int32_t restart;                /* 1 */
  int32_t fixed_iteration_mode;   /* 0 */
  int32_t cr_iters;               /* 9 */
  double baumgarte_beta;          /* 0.2 */
  double contact_margin;          /* 0.01 */
  double impact_velocity_threshold; /* 0.1 */
  double bias_clamp;              /* 10 */
  double limit_margin_angular;    /* 0.01 */
  double limit_margin_linear;     /* 0.001 */
  int32_t warm_start;             /* 1 */
} kd_step_config;

/* Fill *cfg with the reference defaults (StepConfig{}, PadmmConfig{}). */
void kd_step_config_default(kd_step_config* cfg);

/* ---- per-world diagnostics (StepDiagnostics stepper.hpp:63-74 + SolveDiagnostics padmm.hpp:19-28) */
typedef struct kd_step_diag {
  int32_t iterations;
  int32_t restarts;
  int32_t converged;
  int32_t cr_breakdown;
  int64_t cr_iterations;
  double r_p, r_d, r_c;
  int32_t n_rows;
  int32_t contact_count;
  int32_t first_contact_row;
  int32_t n_limits;
  double f_inf;
  double kkt_momentum_inf;
  double bilateral_velocity_inf;
} kd_step_diag;

/* ---- model ------------------------------------------------------------------ */
typedef struct kd_model kd_model;

typedef struct kd_model_info {
  int32_t n_bodies;
  int32_t n_joints;
  int32_t n_geoms;
  int32_t n_bilateral_rows;   /* MechanismModel::n_bilateral_rows (model.hpp:105) */
  int32_t n_dynamics_rows;    /* model.hpp:106 */
  int32_t n_loops;            /* model.hpp:107 */
  int32_t n_limited_joints;
  int32_t max_contacts;       /* capacity: 1 per sphere pair, 4 per box-plane pair */
  int32_t row_capacity;       /* n_bil + n_dyn + 2 n_limited + 3 max_contacts */
} kd_model_info;

/* build_model (model.hpp:117, model.cpp:100-307): validates, lays out rows,
 * counts loops, resolves default PD targets.  On error returns the ModelError
 * code (KD_ERR_MODEL_*) and kd_last_error() holds the reference message. */
int kd_model_build(const kd_scene_desc* scene, kd_model** out);

/* Opt-in extensions beyond the reference (no reference counterpart; parity
 * unpinned).  KD_EXT_BOX_BOX: box-box geom pairs collide (SAT + face clipping,
 * up to 4 contacts per pair) instead of failing with
 * KD_ERR_MODEL_UNSUPPORTED_COLLISION_PAIR (model.cpp:56-62).
 * kd_model_build(scene, out) == kd_model_build_ex(scene, 0, out). */
#define KD_EXT_BOX_BOX 1u
int kd_model_build_ex(const kd_scene_desc* scene, uint32_t extensions, kd_model** out);
void kd_model_destroy(kd_model* model);
/* Contacts a world of this model can hold per step (batches created after the
 * call).  Default: min(max_contacts, 6 n_geoms + 16), 8 n_geoms + 16 with
 * box-box pairs.  The reference's collide() is unbounded (contacts.cpp:119-145)
 * but can never produce more than kd_model_info.max_contacts (1 per sphere
 * pair, 4 per box pair), so capacity = max_contacts reproduces it exactly at
 * the cost of row storage.  A step whose contacts overflow the capacity
 * returns KD_ERR_CAPACITY from kd_batch_step / kd_batch_sync; the overflowing
 * world's state and caches are left unchanged, the other worlds step.
 * capacity <= 0 restores the default; larger values are clamped to max_contacts. */
int kd_model_set_contact_capacity(kd_model* model, int32_t capacity);
int kd_model_get_info(const kd_model* model, kd_model_info* out);
/* JointLayout (model.hpp:63-74): per joint row_offset,row_count,dyn_offset,dyn_count */
int kd_model_joint_layout(const kd_model* model, int32_t* row_offset, int32_t* row_count,
                          int32_t* dyn_offset, int32_t* dyn_count);
/* Resolved per-joint PD targets (JointSpec::target, model.cpp:293-305). */
int kd_model_joint_targets(const kd_model* model, double* targets);
/* joint_coordinate (model.hpp:130, model.cpp:326-340) on host; poses are 7/body. */
int kd_joint_coordinate(const kd_model* model, int32_t joint, const double* poses7, double* out);

/* ---- batch (WorldBatch batch.hpp:14-54, batch_step batch.hpp:58) ------------- */
typedef struct kd_batch kd_batch;

/* Creates a device-resident batch on CUDA device `device`; world w uses
 * models[world_model[w]] and starts from that model's initial state
 * (WorldBatch::add_world(model), batch.cpp:8-11). */
int kd_batch_create(int32_t device, const kd_model* const* models, int32_t n_models,
                    const int32_t* world_model, int32_t n_worlds, kd_batch** out);
void kd_batch_destroy(kd_batch* batch);
int kd_batch_size(const kd_batch* batch, int32_t* n_worlds, int64_t* pose_len, int64_t* twist_len);
/* pose_offset / twist_offset (batch.hpp:31-32) for every world. */
int kd_batch_offsets(const kd_batch* batch, int32_t* pose_offset, int32_t* twist_offset);
/* Whole-batch host<->device state copies in the reference storage layout
 * (pose_storage/twist_storage, batch.hpp:33-34; extract/insert_state batch.cpp:27-72).
 * `time` has one entry per world; any pointer may be NULL to skip that field. */
int kd_batch_set_state(kd_batch* batch, const double* poses, const double* twists, const double* time);
int kd_batch_get_state(kd_batch* batch, double* poses, double* twists, double* time);
/* Clear every warm-start cache (WorldState caches, stepper.hpp:38-56). */
int kd_batch_reset_caches(kd_batch* batch);
/* set_active (batch.hpp:25): one byte per world. */
int kd_batch_set_active(kd_batch* batch, const uint8_t* active);
/* batch_step (batch.hpp:58, batch.cpp:74-110) applied n_steps times on the
 * device stream; returns after the work is enqueued AND completed. */
int kd_batch_step(kd_batch* batch, const kd_step_config* cfg, int32_t n_steps);
/* Asynchronous variant: enqueue n_steps on the batch's CUDA stream and return
 * without synchronising; kd_batch_sync waits and reports device-side errors
 * (SPD failure / capacity overflow).  kd_batch_stream exposes the stream
 * (a cudaStream_t) so callers can record CUDA events around the work. */
int kd_batch_step_async(kd_batch* batch, const kd_step_config* cfg, int32_t n_steps);
int kd_batch_sync(kd_batch* batch);
int kd_batch_stream(kd_batch* batch, void** stream);
/* Zero-copy access to the device-resident state: device
 * pointers to the pose (7 doubles per body) and twist (6 per body) storage in
 * the WorldBatch layout (batch.hpp:41-42) and to the per-world time.  They
 * stay valid for the batch's lifetime; work on them must be ordered with the
 * batch stream (kd_batch_stream). */
int kd_batch_device_state(kd_batch* batch, double** poses, double** twists, double** time);

/* Batched forward kinematics on the device (fk_solve, fk.hpp:33; SURVEY §8f
 * rank 2): for every active world, Gauss-Newton with Levenberg damping on
 * [bilateral f; coordinate - target] from the world's current poses, which
 * are overwritten with the result (twists and time untouched).  joints /
 * values are n_worlds x n_targets (joint index, target coordinate) per world;
 * tolerance / max_iters / lm_initial are FkConfig (fk.hpp:19-23).  Per-world
 * outputs (each may be NULL): iterations, residual_inf, converged.  Any model
 * size: the normal matrix lives in shared memory when it fits (<= 36 bodies),
 * else in a per-world HBM scratch slab (KD_ERR_CAPACITY only if that slab does
 * not fit device memory). */
int kd_batch_fk(kd_batch* batch, const int32_t* joints, const double* values, int32_t n_targets, double tolerance,
                int32_t max_iters, double lm_initial, int32_t* iterations, double* residual_inf, uint8_t* converged);
/* Async state copies with caller-provided (pinned) host buffers, on the batch stream. */
int kd_batch_set_state_async(kd_batch* batch, const double* poses, const double* twists);
int kd_batch_get_state_async(kd_batch* batch, double* poses, double* twists);
/* diagnostics(w)/converged(w) (batch.hpp:27-29) of the last step, per world. */
int kd_batch_get_diagnostics(kd_batch* batch, kd_step_diag* per_world);
/* StepDiagnostics::impulses (stepper.hpp:68) of the last step: world w's rows
 * are written at out[offsets[w] .. offsets[w]+n_rows(w)), offsets[] being the
 * per-world row capacity prefix sum returned by kd_batch_row_offsets. */
int kd_batch_row_offsets(const kd_batch* batch, int64_t* row_offset, int64_t* total_rows);
int kd_batch_get_impulses(kd_batch* batch, double* out);
/* Per-iteration combined residual max(r_p,r_d,r_c) of the last step
 * (padmm_solve combined_history, padmm.hpp:64-67).  Enable with capacity > 0
 * before stepping; out is [n_worlds][capacity], unused tail = -1. */
int kd_batch_set_history_capacity(kd_batch* batch, int32_t capacity);
int kd_batch_get_history(kd_batch* batch, double* out);

/* ---- warm-start caches (WorldState caches, stepper.hpp:38-56; contacts.hpp:32-38) */
/* LimitReactionCache entry: key (joint, bound) -> (lambda, z), physical scale. */
typedef struct kd_limit_cache_entry {
  int32_t joint, bound;
  double lambda, z;
} kd_limit_cache_entry;
/* ReactionCacheEntry (contacts.hpp:32-38): impulse and dual in the contact frame. */
typedef struct kd_contact_cache_entry {
  int32_t geom_a, geom_b;
  double position[3];
  double impulse[3];
  double dual[3];
} kd_contact_cache_entry;
/* Sizes of world w's caches: joint_len = n_bilateral + n_dynamics rows,
 * joint_valid (JointReactionCache::valid), the number of limit entries and of
 * contact entries. */
int kd_batch_get_cache_sizes(kd_batch* batch, int32_t world, int32_t* joint_len, int32_t* joint_valid,
                             int32_t* n_limits, int32_t* n_contacts);
/* extract_state's cache part (batch.cpp:42-44): joint lambda / z (joint_len
 * doubles each), limit entries in (joint, bound) order (std::map order) and
 * contact entries in contact order.  Capacities too small -> KD_ERR_CAPACITY. */
int kd_batch_get_caches(kd_batch* batch, int32_t world, double* joint_lambda, double* joint_z,
                        int32_t* joint_valid, kd_limit_cache_entry* limits, int32_t limit_capacity,
                        int32_t* n_limits, kd_contact_cache_entry* contacts, int32_t contact_capacity,
                        int32_t* n_contacts);
/* insert_state's cache part (batch.cpp:68-70).  The joint cache is used only
 * if joint_len equals the world's n_bilateral + n_dynamics (gather_warmstart,
 * stepper.cpp:25).  Limit keys of joints without limits and contact entries
 * whose (geom_a, geom_b) is not a collision pair of the model can never match
 * a row, so they are dropped.  More contact entries than the world's contact
 * capacity -> KD_ERR_CAPACITY. */
int kd_batch_set_caches(kd_batch* batch, int32_t world, const double* joint_lambda, const double* joint_z,
                        int32_t joint_len, int32_t joint_valid, const kd_limit_cache_entry* limits,
                        int32_t n_limits, const kd_contact_cache_entry* contacts, int32_t n_contacts);

/* ---- solver-level entry points (unit parity on pre-assembled systems) -------- */
/* One pre-assembled system: ConstraintSet (constraints.hpp:39-65: rows in the
 * order bilateral + joint-dynamics | limits | contacts, so the cone product is
 * one Bilateral group, one Nonnegative(1) group per limit row and one
 * SecondOrder(3, mu) group per contact), the per-body inverse mass data of
 * world_inertias (BodyInertiaWorld, delassus.hpp:13-18) and the
 * Preconditioner scale (delassus.hpp:26-29).  All arrays are caller-owned. */
typedef struct kd_solve_problem {
  int32_t n_rows;
  int32_t n_bodies;
  int32_t n_bilateral;        /* rows in the leading Bilateral group */
  int32_t n_limits;           /* Nonnegative rows that follow */
  int32_t n_contacts;         /* SOC triples that follow (3 rows each) */
  int32_t pad;
  const int32_t* body;        /* 2 per row: body_a, body_b (-1: none) */
  const double* jacobian;     /* 12 per row: block_a[6], block_b[6] ([linear; angular]) */
  const double* reg;          /* n_rows: R */
  const double* scale;        /* n_rows: P */
  const double* mu;           /* n_contacts friction coefficients (may be NULL if none) */
  const double* inv_mass;     /* n_bodies */
  const double* inv_inertia;  /* 9 per body, world frame, row-major */
  const double* rhs;          /* n_rows: padmm_solve's v_f (preconditioned), or cr_solve's rhs */
  const double* x0;           /* n_rows or NULL: PadmmInit::x0 / cr_solve's warm start x */
  const double* z0;           /* n_rows or NULL: PadmmInit::z0 */
} kd_solve_problem;

/* build_backend + padmm_solve (delassus.hpp:103-105, padmm.hpp:64-67) for a
 * batch of systems on device `device`: backend Dense (any n, the dense
 * kernel: assembly + Cholesky + PADMM), MatrixFree (the CR kernels, cr_budget
 * per solve) or Auto (Dense iff n <= 300, delassus.cpp:204-206); the operator
 * is D = P (J M^-1 J^T + R) P + eta_rho I.  cfg supplies PadmmConfig (eta,
 * rho, eps, max_iters, acceleration, restart, fixed_iteration_mode); other
 * fields are ignored.  Problem p's lambda (PadmmResult::lambda, preconditioned
 * y) and z go to lambda[off_p..], z[off_p..] with off_p the prefix sum of
 * n_rows; diags[p] gets SolveDiagnostics (iterations, restarts, converged,
 * r_p, r_d, r_c, cr_iterations, cr_breakdown) and n_rows.  history (may be
 * NULL) is [n_problems][history_capacity]: the combined residual per
 * iteration, -1 after the last.  A non-SPD dense system -> KD_ERR_SPD_FAILURE
 * (the reference's runtime_error, delassus.cpp:209-215). */
int kd_padmm_solve_batched(int32_t device, const kd_solve_problem* problems, int32_t n_problems, double eta_rho,
                           int32_t backend, int32_t cr_budget, const kd_step_config* cfg, double* lambda,
                           double* z, kd_step_diag* diags, double* history, int32_t history_capacity);
/* cr_solve(bake_jacobian(cs, inertias, precond, eta_rho), rhs, x, max_iters,
 * &history) (delassus.hpp:82-83, delassus.cpp:130-187) per problem: x0 is
 * the warm start (NULL: zeros), x[off_p..] the result; iterations,
 * breakdown (CrResult::breakdown, raw) and residual_norm per problem (each
 * may be NULL); history (may be NULL): [n_problems][history_capacity] of
 * |r| (initial, then after every update), -1 after the last. */
int kd_cr_solve_batched(int32_t device, const kd_solve_problem* problems, int32_t n_problems, double eta_rho,
                        int32_t max_iters, double* x, int32_t* iterations, uint8_t* breakdown, double* residual_norm,
                        double* history, int32_t history_capacity);
/* assemble_constraints (constraints.hpp:91-94) for every active world of the
 * batch at its current state: runs the device assembly (collide, rows,
 * preconditioner, warm start) without solving or integrating; the rows,
 * contacts and limit keys are then readable with kd_batch_dump_* and
 * kd_batch_get_diagnostics (n_rows, contact_count, n_limits). */
int kd_batch_assemble(kd_batch* batch, const kd_step_config* cfg);

/* ---- one-step introspection for parity (ConstraintSet constraints.hpp:39-65) -- */
typedef struct kd_row_dump {
  int32_t body_a, body_b;
  int32_t kind;        /* 0 bilateral/dynamics, 1 limit (nonnegative), 2 contact (SOC) */
  int32_t pad;
  double block_a[6], block_b[6];
  double bias, reg, scale, vf_scaled, lambda, z;
} kd_row_dump;
/* Rows assembled by the last step of world w (n_rows entries). */
int kd_batch_dump_rows(kd_batch* batch, int32_t world, kd_row_dump* out, int32_t capacity,
                       int32_t* n_rows);
/* Contacts of the last step of world w: geom_a, geom_b per contact and
 * position/normal/depth/mu/e (ContactPoint, contacts.hpp:11-19). */
int kd_batch_dump_contacts(kd_batch* batch, int32_t world, int32_t* geoms, double* data9,
                           int32_t capacity, int32_t* n_contacts);
/* Active limit keys (joint, bound) of the last step (ConstraintSet::limit_keys). */
int kd_batch_dump_limits(kd_batch* batch, int32_t world, int32_t* keys2, int32_t capacity,
                         int32_t* n_limits);

/* ---- multi-GPU helpers --------------------------------------------------------- */
/* Deterministic bench jitter (main.cpp:199-211): std::mt19937_64(seed) +
 * std::normal_distribution<double>(0, sigma), applied world-major, per body,
 * for k=0..2 linear[k] then angular[k].  twists6 is the batch twist storage. */
int kd_bench_jitter(uint64_t seed, double sigma, int32_t n_worlds, const int32_t* n_bodies,
                    double* twists6);

/* Device timing of the last kd_batch_step call, per kernel family:
 * ms[0]=assemble, ms[1]=dense solve, ms[2]=matrix-free solve, ms[3]=recover. */
int kd_batch_enable_timing(kd_batch* batch, int32_t enable);
int kd_batch_get_timing(kd_batch* batch, double* ms4, int64_t* launches);

/* Diagnostics: clock64() cycles of the fused dense kernel's phases for the last
 * step, out[w*8 + k]: 0 scaled Gram assembly, 1 unused, 2 Cholesky, 3 L^{-1},
 * 4 PADMM loop, 5/6/7 Cholesky panel/trailing/diagonal-chain sub-totals
 * (worlds on another backend report zeros). */
int kd_batch_get_phase_cycles(kd_batch* batch, int64_t* out);
/* Diagnostics: which device kernel solved each world's last step:
 * KD_KERNEL_NONE (inactive / no rows), KD_KERNEL_DENSE (fused dense LLT, shared
 * or global factor), KD_KERNEL_SUPERNODAL (sparse LLT with the model's plan),
 * KD_KERNEL_SUPERNODAL_DENSE (the plan's sparse factor, then the dense kernel),
 * KD_KERNEL_CR (matrix-free Conjugate Residual). */
#define KD_KERNEL_NONE 0
#define KD_KERNEL_DENSE 1
#define KD_KERNEL_SUPERNODAL 2
#define KD_KERNEL_CR 3
#define KD_KERNEL_SUPERNODAL_DENSE 4 /* supernodal factor handed to the dense kernel's L^{-1} + solves */
#define KD_KERNEL_SUPERNODAL_CLUSTER 5 /* as 4, with the PADMM solves on a CTA pair (K2c, opt-in: KD_CLUSTER=1) */
int kd_batch_get_kernels(kd_batch* batch, int32_t* out);

/* Per world, which matrix-free kernel solved the last step (diagnostics; the
 * three compute the same cr_solve / MatrixFreeDelassus::apply, delassus.cpp:
 * 106-187): KD_CR_PATH_NONE (not on the matrix-free backend),
 * KD_CR_PATH_INCIDENCE (incidence-owner lanes keep P J in registers),
 * KD_CR_PATH_ROWS (row owners keep P J in registers), KD_CR_PATH_SHARED
 * (P J staged in shared memory or streamed; worlds above 1024 rows; worlds
 * whose vectors exceed one CTA's shared memory keep them in a per-world HBM
 * slab, so there is no size limit). */
#define KD_CR_PATH_NONE 0
#define KD_CR_PATH_INCIDENCE 1
#define KD_CR_PATH_ROWS 2
#define KD_CR_PATH_SHARED 3
int kd_batch_get_cr_paths(kd_batch* batch, int32_t* out);

/* Supernodal sparse-LLT plan of a model (the factorization the device uses for
 * the reference's Dense backend, DenseDelassus delassus.cpp:59-65, on models
 * whose static row-capacity pattern admits one).  stats[0..11] = slots S,
 * nnz(L), per-world fp64 array length, supernodes, solve levels, solve
 * program words, factor FMAs, solve FMA terms per PADMM iteration, dense-LLT
 * FMAs S^3/6, per-world shared-memory doubles, solve critical path (terms on
 * the busiest lane, summed over phases), solve phases, and the 64-bit masks of
 * the nonzero 32x32 tiles of L and of L^-1 (bit ti(ti+1)/2 + tj).
 * Returns KD_ERR_INVALID_ARGUMENT with the reason if the model has no plan. */
int kd_model_sparse_plan_info(const kd_model* model, int64_t* stats14);
/* Host self-test of the plan (no device): a random SPD system with the plan's
 * pattern and a random active-slot mask, solved by the plan's factor and solve
 * programs and by a dense Cholesky; writes the max relative difference. */
int kd_model_sparse_plan_selftest(const kd_model* model, uint64_t seed, double* max_rel_err);

const char* kd_last_error(void);
const char* kd_version(void);
/* ABI self-check: writes sizeof of kd_body_desc, kd_joint_desc, kd_geom_desc,
 * kd_scene_desc, kd_step_config, kd_step_diag, kd_model_info, kd_row_dump,
 * kd_limit_cache_entry and kd_contact_cache_entry, in that order, into
 * out[0..9]; returns the count written (at most capacity). */
int kd_abi_sizes(int32_t* out, int32_t capacity);

#ifdef __cplusplus
}
#endif
#endif /* KAMINO_B200_H */
