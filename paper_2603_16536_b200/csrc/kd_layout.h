// kd_layout.h — HBM data layout of a device-resident world batch.
//
// Model data (immutable, shared by all worlds of a model; L2/L1-resident):
//   DevModel (one per model) indexes arrays of DevBody / DevJoint / DevGeom /
//   DevPair.  These are the reference MechanismModel (model.hpp:97-113) with
//   the row layout (JointLayout, model.hpp:63-74), frame rotations and the
//   ordered collision-pair list (contacts.cpp:119-145) precomputed on the host.
//
// World state (the WorldBatch storage, batch.hpp:41-42): poses7 / twists6 in the
//   reference AoS-per-world layout with prefix-sum offsets, so host<->device
//   copies are single memcpys and a CTA/warp reads one contiguous slab.
//
// Per-step scratch (SoA over rows / bodies / contacts, each world owning a
//   capacity-sized slab at a prefix-sum offset): rows are addressed
//   row_off[w] + r with r in the reference row order
//   [bilateral | dynamics | limits | contacts] (constraints.hpp:33-38).
#pragma once
#include <cstddef>

#include <stdint.h>

namespace kd {

enum JointKind : int32_t { J_FIXED = 0, J_REVOLUTE = 1, J_PRISMATIC = 2, J_SPHERICAL = 3 };
enum GeomShape : int32_t { G_SPHERE = 0, G_PLANE = 1, G_BOX = 2 };
// Collision pair kinds in collide() dispatch order (contacts.cpp:130-140);
// `a` is always the moving geom (ContactPoint::geom_a), `b` the other one.
enum PairKind : int32_t { P_SPHERE_SPHERE = 0, P_SPHERE_PLANE = 1, P_BOX_PLANE = 2, P_BOX_BOX = 3 };
enum RowKind : int32_t { ROW_BILATERAL = 0, ROW_LIMIT = 1, ROW_CONTACT = 2 };
// BE_DENSE_SN: the supernodal kernel factors (plan order) and hands L to the
// dense kernel, which forms L^-1 and runs the PADMM solves
enum Backend : int32_t {
  BE_NONE = -1,
  BE_DENSE_SMEM = 0,
  BE_DENSE_GLOBAL = 1,
  BE_MATRIX_FREE = 2,
  BE_SPARSE = 3,
  BE_DENSE_SN = 4,
};

enum JointFlags : int32_t {
  JF_PD = 1,
  JF_ARMATURE = 2,
  JF_DAMPING = 4,
  JF_LIMITS = 8,
};

struct DevBody {
  double mass, inv_mass;
  double ib[9];  // body-frame inertia
};

struct DevJoint {
  int32_t type, parent, child, flags;
  int32_t row_offset, row_count, dyn_offset, limit_slot;  // limit_slot: index among limited joints
  double fp_pos[3], fc_pos[3];
  double fp_q[4], fc_q[4];     // frame orientations [w,x,y,z]
  double fp_R[9], fc_R[9];     // Eigen toRotationMatrix of the frame orientations
  double axis[3], comp0[3], comp1[3];
  double lower, upper, kp, kd, target, target_rate, armature, damping;
};

struct DevGeom {
  int32_t body, shape, pad0, pad1;
  double radius, he[3], normal[3], offset, mu, restitution;
};

struct DevPair {
  int32_t a, b, kind, pad;
};

struct DevModel {
  int32_t nb, nj, ng, npairs;
  int32_t n_bil, n_dyn, n_limited, max_contacts;
  int32_t row_cap, body_off, joint_off, geom_off;
  int32_t pair_off, sn, pad1, pad2;  // sn: 1 supernodal kernel, 2 supernodal factor + dense solve
  double gravity[3];
  double pad3;
};

// ---- supernodal sparse-LLT plan (kd_snplan.h), one per model, immutable.
// D entry of the Gram phase: D(s, t), s >= t (slot order).
struct SnGram {
  uint16_t dst;  // Lv index
  uint16_t s, t; // slots
  uint16_t flags;
};
enum SnGramFlags : uint16_t {
  SG_DIAG = 1,
  SG_TWO = 2,  // two shared bodies
  SG_S1 = 4,   // side of s for the first (smaller) shared body
  SG_T1 = 8,   // side of t for the first shared body
  SG_S2 = 16,  // sides for the second shared body
  SG_T2 = 32,
};
// Gram by body (ascending): the k rows touching the body (slot | side << 16 at
// gslot[slot_off..]) are staged, then its n_store + n_acc pairs (Lv index |
// local i << 16 | local j << 24 at gpair[pair_off..]) are written / added.
struct SnGBody {
  int32_t slot_off, k, pair_off, n_store;
  int32_t n_acc, pad0, pad1, pad2;
};
// One supernode: columns [c0, c0+w) of the factor in elimination order, with
// m rows below the diagonal block.  Its dense panel ((w+m) x w, column-major,
// odd column stride ld) lives at Lv[pb]; rows 0..w-1 are the supernode's own
// positions, rows w.. its row structure.  X = L_SS^-1 (w x w, row stride ws)
// lives at Lv[xb]; X's diagonal holds 1/L_jj.  The right-looking update of the
// ancestors reads m(m+1)/2 target entries at tmap[tmap_off..]:
// Lv index | ri << 16 | rj << 24.
struct SnSuper {
  int32_t c0, w, m, ld;
  int32_t pb, xb, ws, tmap_off;
  int32_t prow_off, pad0, pad1, pad2;  // w + m panel-row positions at sn_prow[prow_off..]
};
// Solve program (one u32 blob per model, copied to shared memory per CTA):
//   phase (4 words): rec0 (word offset of its records), nsteps, mode, split
//   record (2 words): dst | nterm << 16 ;  toff (word offset of the chunk's
//     terms) | npart << 24 | owner << 30 | valid << 31
//   term (1 word): Lv index | vector index << 16
// mode 0 (A): t[dst] = v[dst] - sum Lv[a] v[b];  mode 1 (B): v[dst] = sum Lv[a] t[b].
// A row's terms may be split over consecutive slots (chunks); its first chunk
// (owner) adds the others' partial sums in slot order after a __syncwarp.
constexpr int kSnChunk = 8;  // max terms per solve chunk (the kernel's unrolled width)
struct DevSnPlan {
  int32_t S, nLv, n_jd, lim_base;
  int32_t gram_off, n_gram, pair_off, slotpos_off;
  int32_t sup_off, n_sup, prog_off, prog_words;
  int32_t n_sph, max_slots, smem_doubles, cl_split;  // smem_doubles: per-warp footprint of K2s; cl_split: first tile row of the cluster PADMM kernel's second CTA (0: the model does not take K2c)
  int32_t gbody_off, n_gbody, kmax, vreg;  // vreg: per-warp vector region (doubles)
  int32_t lmask_lo, lmask_hi, scat_off, n_scat;  // nonzero 32x32 tiles of L in plan order; hand-off scatter list
  int32_t xmask_lo, xmask_hi, kmask_off, cl_xlen;  // nonzero 32x32 tiles of L^-1; per-L-tile column-group masks; K2c slab doubles per world
};

// Per-world indexing (prefix sums over model capacities).
struct DevWorld {
  int32_t model, nb, pose_off, twist_off;
  int64_t row_off;      // rows (capacity n_bil + n_dyn + 2 n_limited + 3 contact_cap)
  int32_t body_off;     // bodies
  int32_t contact_off;  // contacts
  int32_t jcache_off;   // n_bil + n_dyn
  int32_t lslot_off;    // 2 * n_limited
  int32_t bin;          // dense-smem bin
  int32_t smem_cap;     // rows the bin's dense-smem kernel can hold
  int32_t contact_cap;  // contacts this world can hold (overflow is reported, never silent)
  int32_t slab_cap;     // rows the dense-global slab can hold (0 if none)
  int64_t lslab_off;    // dense-global factor slab (doubles), -1 if none
  int64_t snlv_off;     // supernodal factor hand-off slab (doubles), -1 if none
  int64_t snr2p_off;    // row -> plan position hand-off (int32), -1 if none
  int64_t xslab_off;    // K2c: the world's X = L^-1 tiles (compact, row-major), -1 if the world does not take K2c
};

// Per-row Jacobian blocks: J = [block_a | block_b], JM = J M^-1 folded
// (fold_inverse_mass, delassus.cpp:12-17).
struct RowJ {
  double J[12];
  double JM[12];
};

// Per-body step scratch.
struct BodyS {
  double ep[3];      // evaluation pose (Moreau-Jean half step)
  double eq[4];
  double eR[9];
  double uf[6];      // u_free
  double h[6];       // free forces at start-of-step poses
  double Iw[9];      // world inertia at eval pose
  double Iwinv[9];
  double mass, inv_mass;
  double up[6];      // u+
};

// K1 moves RowJ halves and BodyS::uf with 16-byte accesses (arrays are cudaMalloc'd)
static_assert(sizeof(RowJ) % 16 == 0, "RowJ rows must keep 16-byte alignment");
static_assert(sizeof(BodyS) % 16 == 0 && offsetof(BodyS, uf) % 16 == 0, "BodyS::uf must be 16-byte aligned");

struct Contact {
  int32_t ga, gb, pair, pad;
  double pos[3], nrm[3];
  double depth, mu, e;
};

struct CacheEntry {
  int32_t ga, gb, pair, pad1;  // pair: index in the model's pair list (the cache is sorted by it)
  double pos[3], imp[3], dual[3];
};

// Per-world step results that are not rows.
struct WorldStep {
  int32_t n_rows, n_limits, n_contacts, backend;
  int32_t iterations, restarts, converged, cr_breakdown;
  int64_t cr_iterations;
  double r_p, r_d, r_c;
  double f_inf, kkt, bil_vel;
  int32_t jcache_valid, ccache_count, fail, cr_path;  // cr_path: 1 if the incidence-owner CR kernel took the world
  int64_t phase_cycles[8];  // fused-kernel phase stamps (clock64 deltas), diagnostics only
};

// Everything a kernel needs, passed by value (device pointers).
struct BatchView {
  int32_t n_worlds;
  int32_t hist_cap;
  const DevModel* models;
  const DevBody* bodies;
  const DevJoint* joints;
  const DevGeom* geoms;
  const DevPair* pairs;
  const DevWorld* worlds;
  const uint8_t* active;
  double* poses;
  double* twists;
  double* time;
  WorldStep* wstep;
  // rows
  RowJ* rowj;
  int32_t* rbody;   // 2 per row
  int32_t* rkind;
  int32_t* lkey;    // 2 per row (joint, bound) for limit rows
  double* rmu;
  double* bias;
  double* reg;
  double* scale;
  double* vf;       // P (J u_free - v*)
  double* x0;
  double* z0;
  double* lam;      // solver y (preconditioned)
  double* zo;       // solver z (preconditioned)
  double* imp;      // physical impulses P y
  int32_t* csr_ptr; // per world nb+1 entries at body_off + world
  int32_t* csr;     // per world 2*row_cap entries at 2*row_off: row*2 + side
  // bodies
  BodyS* bs;
  // contacts + caches
  Contact* contacts;
  CacheEntry* ccache;
  double* jc_lam;
  double* jc_z;
  double* ls_lam;
  double* ls_z;
  int32_t* ls_valid;
  double* lslab;    // dense-global factor storage
  double* hist;     // [n_worlds][hist_cap]
  int32_t* error_count;
  // supernodal plans (indexed by model; S == 0: none)
  const DevSnPlan* snplan;
  const SnGram* sn_gram;
  const SnGBody* sn_gbody;
  const uint32_t* sn_gslot;
  const uint32_t* sn_gpair;
  const SnSuper* sn_sup;
  const uint32_t* sn_tmap;
  const uint32_t* sn_prog;
  const int32_t* sn_pair_slot;
  const uint16_t* sn_slot_pos;
  const int32_t* sn_prow;  // panel-row positions of every supernode
  const uint32_t* sn_scat; // hand-off scatter lists (Lv index | tile index << 16)
  const uint8_t* sn_kmask;  // per-L-tile 4-column-group nonzero masks (36 per planned model)
  double* cr_scratch;      // worlds too large for one CTA's shared memory: the shared CR kernel's
  int64_t cr_scratch_stride;  // per-world HBM slab (doubles per world, indexed by world), else null
  double* xslab;           // K2c hand-off: X = L^-1 per world (nonzero tiles, row-major; off-diagonal 32 x 33, diagonal 528)
  double* sn_lv;           // BE_DENSE_SN hand-off: the factor array per world
  int32_t* sn_r2p;         // BE_DENSE_SN hand-off: compact row -> position per world
};

struct StepParams {
  double dt, eta, rho, eps;
  double beta, contact_margin, impact_thr, bias_clamp, lim_margin_ang, lim_margin_lin;
  int32_t max_iters, acceleration, restart, fixed_mode;
  int32_t cr_iters, warm_start, moreau, backend;  // backend: KD_BACKEND_*
  int32_t sparse, sn_handoff;                      // supernodal path enabled / factor hand-off enabled
  int32_t cr_only, no_df, no_tmem;  // no_tmem: KD_TMEM=0 (dense solve tiles from shared memory, not tensor memory); no_df: KD_DENSE_DF=0 (dense solve passes with a barrier, not dataflow flags); cr_only: one cr_solve(op, rhs = vf, x = x0, cr_iters) per world, no PADMM (kd_cr_solve_batched)
  double eta_rho;         // the operator's eta + rho (build_backend's argument; eta + rho in a step)
  const double* nest_beta;  // Nesterov beta_m = (a_m - 1) / a_{m+1}, a_0 = 1, m < max_iters (padmm.cpp:54-71)
};

}  // namespace kd
