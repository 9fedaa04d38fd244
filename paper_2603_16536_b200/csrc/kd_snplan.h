// kd_snplan.h — per-model symbolic plan of the supernodal sparse LLT path.
//
// The reference factors the preconditioned Delassus matrix densely
// (DenseDelassus, Eigen LLT<MatrixXd>, delassus.cpp:59-65).  D is block
// sparse: D_ij != 0 only when rows i and j share a body (assemble_dense sums
// per-body Gram blocks, delassus.cpp:67-104).  For a mechanism model the set of
// rows that can exist is static — the model's row capacity
//   [bilateral | dynamics | 2 slots per limited joint | 3 per potential contact]
// (model.cpp:254-276; the limit/contact slots are the ones K1 may activate) —
// so the sparsity pattern, a fill-reducing ordering, the symbolic factor and a
// level-scheduled instruction stream for the numeric factor and the two
// triangular solves are computed once per model on the host.  Inactive slots
// become identity rows (D_ss = 1, zero coupling, zero right-hand side), which
// leaves the active system's solution unchanged.
//
// Device programs (all indices are 16-bit offsets into one per-world fp64
// array `Lv` or into the slot-position vectors):
//   factor:  op {dst, aux, terms (a,b)}:   acc = Lv[dst] - sum Lv[a]*Lv[b]
//            OFF:  Lv[dst] = acc * Lv[aux]        (aux = 1/L_jj)
//            DIAG: Lv[dst] = 1/sqrt(acc)          (the diagonal is only ever
//                                                  used as its reciprocal)
//            The inverse X = L_SS^-1 of every supernode's diagonal block is
//            produced by OFF ops too (X_ij = -(sum_k L_ik X_kj) / L_ii).
//   solve:   phase A: t[dst] = v[dst] - sum Lv[a]*v[b]     (off-block rows/cols)
//            phase B: v[dst] = sum Lv[a]*t[b]              (X or X^T of a block)
//            forward over supernode levels leaves->root, backward root->leaves.
// Ops of one level are independent; they are packed onto 32 lanes (longest
// processing time first) and laid out [step][lane] so a warp reads them
// coalesced.
#pragma once

#include <stdint.h>

#include <string>
#include <vector>

#include "kd_layout.h"

namespace kd {

struct HostModel;

struct SnPlanHost {
  int S = 0;         // planned slots (static rows, limit slots, body-world contact slots)
  int nLv = 0;       // fp64 entries of the per-world factor array
  int smem_doubles = 0;  // per-warp shared-memory footprint of the device kernel
  int n_jd = 0;      // static rows (bilateral + dynamics): slot == row
  int lim_base = 0;  // first limit slot (2 per limited joint: lower, upper)
  std::vector<int32_t> pair_slot;   // per collision pair: first contact slot, -1 if unplanned
  std::vector<uint16_t> slot_pos;   // slot -> elimination position
  std::vector<int32_t> slot_body;   // 2 per slot: (body a, body b or -1)
  std::vector<SnGram> gram;
  std::vector<SnPhase> fphase;
  std::vector<SnOp> fops;
  std::vector<uint32_t> fterms;     // a | b << 16
  std::vector<SnPhase> sphase;
  std::vector<SnSOp> sops;
  std::vector<uint32_t> sterms;     // Lv index | vector index << 16
  // statistics
  int nnzL = 0, n_super = 0, s_levels = 0;
  int64_t factor_terms = 0, solve_terms = 0, dense_factor_terms = 0;
  int factor_crit = 0, solve_crit = 0;  // per-lane critical path (terms + ops)
};

// Builds the plan; returns false (with a reason) if the model is not suited
// (too many slots for 16-bit indices or the per-world array too large).
bool build_sn_plan(const HostModel& m, SnPlanHost& p, std::string& why);

// CPU interpreter of a plan (self-test only): factor the SPD matrix given as a
// dense row-major S x S array (only the plan's pattern is read; `active`
// marks live slots, others become identity rows) and solve D x = b.  Returns
// false on a non-positive pivot.  Vectors are in slot order.
bool sn_plan_cpu_solve(const SnPlanHost& p, const double* D, const uint8_t* active, const double* b, double* x);

}  // namespace kd
