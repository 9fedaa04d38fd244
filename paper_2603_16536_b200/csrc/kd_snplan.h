// kd_snplan.h — per-model symbolic plan of the supernodal sparse LLT path.
//
// The reference factors the preconditioned Delassus matrix densely
// (DenseDelassus, Eigen LLT<MatrixXd>, delassus.cpp:59-65).  D is block
// sparse: D_ij != 0 only when rows i and j share a body (assemble_dense sums
// per-body Gram blocks, delassus.cpp:67-104).  For a mechanism model the set of
// rows that can exist is static — its static rows, both bounds of every
// limited joint, and the contact slots of its body-world collision pairs
// (model.cpp:254-276; K1 activates limits and contacts into those slots) — so
// the sparsity pattern, a fill-reducing ordering, the supernode partition and
// the triangular-solve program are computed once per model on the host.
// Inactive slots become identity rows (D_ss = 1, zero coupling, zero
// right-hand side), which leaves the active system's solution unchanged.
//
// Device execution (kd_sparse.cu, one warp per world):
//   factor: supernodes in postorder; dense right-looking Cholesky of each
//           supernode's panel, X = L_SS^-1 of its diagonal block, then the
//           update of its ancestors through a precomputed target map
//           (sequential over supernodes, so every entry is accumulated in one
//           fixed order);
//   solve:  forward (leaves -> root) then backward, two phases per supernode
//           level: A = off-block dot products, B = X or X^T of the blocks.
//           Phases are packed onto the 32 lanes with long rows split into
//           chunks (owner lane combines), and the whole program is copied to
//           shared memory once per CTA.
#pragma once

#include <stdint.h>

#include <string>
#include <vector>

#include "kd_layout.h"

namespace kd {

struct HostModel;

struct SnPlanHost {
  int S = 0;             // planned slots (static rows, limit slots, body-world contact slots)
  int nLv = 0;           // fp64 entries of the per-world factor array (panels + X blocks)
  int n_jd = 0;          // static rows (bilateral + dynamics): slot == row
  int lim_base = 0;      // first limit slot (2 per limited joint: lower, upper)
  int smem_doubles = 0;  // per-warp shared-memory footprint of the device kernel
  int max_slots = 0;     // largest phase (slots) of the solve program
  int n_sph = 0;         // solve phases
  int kmax = 0;          // most rows touching one body
  int vreg = 0;          // per-warp vector region (doubles)
  uint64_t lmask = 0;      // nonzero 32x32 tiles of L (tile ti(ti+1)/2 + tj), for S <= 256
  uint64_t xmask = 0;      // nonzero 32x32 tiles of X = L^-1 (same numbering)
  std::vector<uint8_t> kmask;  // per L tile (same numbering, S <= 256): 4-column groups with a nonzero
  std::vector<int32_t> pair_slot;   // per collision pair: first contact slot, -1 if unplanned
  std::vector<uint16_t> slot_pos;   // slot -> elimination position
  std::vector<int32_t> slot_body;   // 2 per slot: (body a, body b or -1)
  std::vector<SnGram> gram;
  std::vector<SnGBody> gbody;       // per body: its rows and Gram pairs
  std::vector<uint32_t> gslot;      // slot | side << 16
  std::vector<uint32_t> gpair;      // Lv index | local row i << 16 | local row j << 24
  std::vector<SnSuper> sup;
  std::vector<uint32_t> tmap;
  std::vector<int32_t> prow;        // per supernode: its w + m panel-row positions
  std::vector<uint32_t> scat;       // hand-off scatter: Lv index | dense tile index (n = S) << 16
  std::vector<uint32_t> prog;       // solve program blob (see kd_layout.h)
  // statistics
  int nnzL = 0, s_levels = 0;
  int64_t factor_fma = 0, solve_terms = 0, dense_factor_fma = 0;
  int solve_crit = 0;  // sum over phases of the heaviest lane (terms)
};

// Builds the plan; returns false (with a reason) if the model is not suited.
bool build_sn_plan(const HostModel& m, SnPlanHost& p, std::string& why);

// CPU interpreter of a plan (self-test only): runs the device algorithm on the
// SPD matrix given as a dense row-major S x S array (only the plan's pattern is
// read; `active` marks live slots, others become identity rows) and solves
// D x = b.  Returns false on a non-positive pivot.  Vectors are in slot order.
bool sn_plan_cpu_solve(const SnPlanHost& p, const double* D, const uint8_t* active, const double* b, double* x);

}  // namespace kd
