// kd_snfactor.cu — K2f: the hand-off factor, one CTA per world.
//
// For a model whose worlds take the hand-off (Backend BE_DENSE_SN, see
// kd_dense.cu), this kernel forms D = P (J M^-1 J^T + R) P + (eta+rho) I
// (assemble_dense, delassus.cpp:67-104) in the fill-reducing order of the
// model's supernodal plan (kd_snplan.h) and factors it, D = L L^T
// (DenseDelassus, delassus.cpp:59-65), supernode by supernode.  The panels
// (with 1/L_jj on their diagonals) and the row -> plan-position map go to HBM;
// the dense kernel scatters them into its tile layout and forms L^-1.
//
// Work split inside the CTA:
//   Gram     one thread per D entry of the plan's pattern: the entry's one or
//            two shared-body products are summed in ascending body order (the
//            reference's per-body accumulation order), then + R, P scaling
//            and + (eta+rho) on the diagonal.
//   factor   supernodes in postorder; warp 0 factors the panel (one row per
//            lane, columns in order), then every thread takes entries of the
//            supernode's ancestor update (each target entry is updated once
//            per supernode, so updates accumulate in postorder, as in the
//            sequential algorithm).
// Shared memory per CTA: Lv[nLv] | P[S] | int16 slot2row[S] | int16 row2pos[S]
// (DR-Legs: 38 KB, five CTAs per SM).
#include "kd_device.cuh"

namespace kd {

namespace {
constexpr int kFactorThreads = 128;
constexpr int kFactorMinBlocks = 5;
__host__ __device__ __forceinline__ int pad2(int x) { return (x + 1) & ~1; }

// Panel factor with the panel in registers (rows <= 32, width <= WMAX <= 24): lane q
// holds row q.  Column c: the pivot comes from lane c, rows below it scale by
// 1/L_cc, then row q's columns j in (c, w) take -= L_qc L_jc with L_jc from
// lane j.  Same operations, operands and order as the shared-memory version
// (one fused multiply-add per update), so the factor is bit-identical.
template <int WMAX>
__device__ __forceinline__ bool panel_factor_reg(double* Pn, int w, int rows, int ld, int lane) {
  bool bad = false;
  double row[WMAX];
#pragma unroll
  for (int c = 0; c < WMAX; ++c) row[c] = (c < w && lane < rows) ? Pn[c * ld + lane] : 0.0;
#pragma unroll
  for (int c = 0; c < WMAX; ++c) {
    if (c < w) {  // warp-uniform
      const double d = __shfl_sync(0xffffffffu, row[c], c);
      if (!(d > 0.0)) bad = true;
      const double r = fast_rsqrt(d);
      row[c] = lane > c ? row[c] * r : (lane == c ? r : row[c]);  // the diagonal keeps 1/L_cc
      // L_jc from lane j: unconditional shuffles (no divergent region), predicated updates
#pragma unroll
      for (int j = c + 1; j < WMAX; ++j) {
        const double ljc = __shfl_sync(0xffffffffu, row[c], j);
        if (j < w && lane >= j) row[j] -= row[c] * ljc;
      }
    }
  }
#pragma unroll
  for (int c = 0; c < WMAX; ++c)
    if (c < w && lane >= c && lane < rows) Pn[c * ld + lane] = row[c];
  return bad;
}

}  // namespace

__global__ void __launch_bounds__(kFactorThreads, kFactorMinBlocks)
    snfactor_kernel(BatchView bv, StepParams sp, const int32_t* worlds) {
  extern __shared__ __align__(16) double smem[];
  constexpr int NT = kFactorThreads;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int w = worlds[blockIdx.x];
  WorldStep& ws = bv.wstep[w];
  if (ws.backend != BE_DENSE_SN) return;
  const DevWorld W = bv.worlds[w];
  const DevSnPlan P = bv.snplan[W.model];
  const DevModel M = bv.models[W.model];
  const int S = P.S, Sp = pad2(S);
  double* Lv = smem;
  double* Ps = Lv + pad2(P.nLv);
  int16_t* slot2row = reinterpret_cast<int16_t*>(Ps + Sp);
  int16_t* row2pos = slot2row + Sp;

  const int64_t R0 = W.row_off;
  const int n = ws.n_rows;
  const int nc = ws.n_contacts;
  const int n_jd = P.n_jd;
  const int first_contact = n_jd + ws.n_limits;
  const uint16_t* slot_pos = bv.sn_slot_pos + P.slotpos_off;

  long long t0 = clock64(), c_panel = 0, c_upd = 0, c_fn = 0;
  // ---- 0. zero the factor, map compact rows <-> planned slots
  for (int e = tid; e < P.nLv; e += NT) Lv[e] = 0.0;
  for (int s = tid; s < S; s += NT) slot2row[s] = s < n_jd ? (int16_t)s : (int16_t)-1;
  for (int r = tid; r < n_jd; r += NT) row2pos[r] = (int16_t)slot_pos[r];
  for (int r = tid; r < n; r += NT) Ps[r] = bv.scale[R0 + r];
  __syncthreads();
  {
    const int32_t* lk = bv.lkey + 2 * R0;
    const DevJoint* mj = bv.joints + M.joint_off;
    for (int r = n_jd + tid; r < first_contact; r += NT) {  // limit rows: (joint, bound) -> slot
      const int slot = P.lim_base + 2 * mj[lk[2 * r]].limit_slot + lk[2 * r + 1];
      slot2row[slot] = (int16_t)r;
      row2pos[r] = (int16_t)slot_pos[slot];
    }
    const Contact* ct = bv.contacts + W.contact_off;
    const int32_t* pslot = bv.sn_pair_slot + P.pair_off;
    for (int c = tid; c < nc; c += NT) {  // contacts: (pair, index within the pair) -> slot
      const int pr = ct[c].pair;
      int k = 0;
      while (c - k - 1 >= 0 && ct[c - k - 1].pair == pr) ++k;
      const int slot = pslot[pr] + 3 * k;
      for (int d = 0; d < 3; ++d) {
        slot2row[slot + d] = (int16_t)(first_contact + 3 * c + d);
        row2pos[first_contact + 3 * c + d] = (int16_t)slot_pos[slot + d];
      }
    }
  }
  __syncthreads();

  // ---- 1. Gram, one thread per entry of the plan's pattern.  D(s, t) =
  // JM_s(b1) . J_t(b1) [+ JM_s(b2) . J_t(b2)], b1 < b2 the shared bodies;
  // inactive slots become identity rows.
  {
    const RowJ* rj = bv.rowj + R0;
    const double* reg = bv.reg + R0;
    const double eta_rho = sp.eta_rho;
    const SnGram* gl = bv.sn_gram + P.gram_off;
    // two entries per thread and pass, so their descriptor and J loads overlap
    auto entry = [&](const SnGram g) {
      const int rs = slot2row[g.s], rt = slot2row[g.t];
      const bool diag = g.flags & SG_DIAG;
      if (rs < 0 || rt < 0) {
        if (diag) Lv[g.dst] = 1.0;
        return;
      }
      // 16-byte loads of the row halves (RowJ rows are 16-byte aligned)
      auto half_dot = [](const double* a, const double* c) {
        const double2* a2 = reinterpret_cast<const double2*>(a);
        const double2* c2 = reinterpret_cast<const double2*>(c);
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double2 x = a2[k], y = c2[k];
          s += x.x * y.x;
          s += x.y * y.y;
        }
        return s;
      };
      double s = half_dot(rj[rs].JM + ((g.flags & SG_S1) ? 6 : 0), rj[rt].J + ((g.flags & SG_T1) ? 6 : 0));
      if (g.flags & SG_TWO)
        s += half_dot(rj[rs].JM + ((g.flags & SG_S2) ? 6 : 0), rj[rt].J + ((g.flags & SG_T2) ? 6 : 0));
      if (diag) s += reg[rs];
      double d = (Ps[rs] * s) * Ps[rt];
      if (diag) d += eta_rho;
      Lv[g.dst] = d;
    };
    for (int e = tid; e < P.n_gram; e += 2 * NT) {
      const SnGram g0 = gl[e];
      const bool two = e + NT < P.n_gram;
      const SnGram g1 = two ? gl[e + NT] : g0;
      entry(g0);
      if (two) entry(g1);
    }
  }
  __syncthreads();

  // ---- 2. supernodal right-looking Cholesky in postorder
  const long long t1 = clock64();
  bool bad = false;
  const SnSuper* sup = bv.sn_sup + P.sup_off;
  SnSuper un = sup[0];
  for (int k = 0; k < P.n_sup; ++k) {
    const long long q0 = clock64();
    const SnSuper u = un;
    if (k + 1 < P.n_sup) un = sup[k + 1];  // next descriptor in flight during this supernode
    double* Pn = Lv + u.pb;
    const int rows = u.w + u.m;
    // this thread's first target-map words, loaded while warp 0 factors the panel
    const int T = u.m * (u.m + 1) / 2;
    const uint32_t* tm = bv.sn_tmap + u.tmap_off;
    constexpr int kTE = 4;
    uint32_t tep[kTE];
#pragma unroll
    for (int i = 0; i < kTE; ++i) tep[i] = tid + i * NT < T ? tm[tid + i * NT] : 0u;
    if (wid == 0 && rows <= 32 && u.w <= 16) {
      const long long f0 = clock64();
      const bool b = u.w <= 8 ? panel_factor_reg<8>(Pn, u.w, rows, u.ld, lane)
                              : panel_factor_reg<16>(Pn, u.w, rows, u.ld, lane);
      bad = bad || b;
      __syncwarp();
      c_fn += clock64() - f0;
    } else if (wid == 0) {
      for (int c = 0; c < u.w; ++c) {
        double* col = Pn + c * u.ld;
        const double d = col[c];
        if (!(d > 0.0)) bad = true;
        const double r = fast_rsqrt(d);
        for (int q = c + 1 + lane; q < rows; q += 32) col[q] *= r;
        __syncwarp();
        if (lane == 0) col[c] = r;  // the dense kernel reads 1/L_cc on the diagonal
        // trailing update of the panel's remaining columns
        for (int q = c + 1 + lane; q < rows; q += 32) {
          const double lq = col[q];
          const int jmax = min(q, u.w - 1);
          int j = c + 1;
          for (; j + 3 <= jmax; j += 4) {  // loads first: the stores cannot alias them
            const double c0 = col[j], c1 = col[j + 1], c2 = col[j + 2], c3 = col[j + 3];
            double* p0 = Pn + j * u.ld + q;
            const double p00 = p0[0], p01 = p0[u.ld], p02 = p0[2 * u.ld], p03 = p0[3 * u.ld];
            p0[0] = p00 - lq * c0;
            p0[u.ld] = p01 - lq * c1;
            p0[2 * u.ld] = p02 - lq * c2;
            p0[3 * u.ld] = p03 - lq * c3;
          }
          for (; j <= jmax; ++j) Pn[j * u.ld + q] -= lq * col[j];
        }
        __syncwarp();
      }
    }
    __syncthreads();
    const long long q1 = clock64();
    // ancestors: A_ij -= sum_c L_ic L_jc for i >= j in the row structure
    if (T > 0) {
      for (int e = tid, i = 0; e < T; e += NT, ++i) {
        uint32_t te = tep[0];
#pragma unroll
        for (int q = 1; q < kTE; ++q)
          if (i == q) te = tep[q];
        if (i >= kTE) te = tm[e];
        const double* a = Pn + u.w + ((te >> 16) & 0xff);
        const double* b = Pn + u.w + (te >> 24);
        double s0 = 0.0, s1 = 0.0;
        int c = 0;
        for (; c + 1 < u.w; c += 2) {
          s0 += a[c * u.ld] * b[c * u.ld];
          s1 += a[(c + 1) * u.ld] * b[(c + 1) * u.ld];
        }
        if (c < u.w) s0 += a[c * u.ld] * b[c * u.ld];
        Lv[te & 0xffff] -= s0 + s1;
      }
      __syncthreads();
    }
    c_panel += q1 - q0;
    c_upd += clock64() - q1;
  }
  if (tid == 0) {
    ws.phase_cycles[5] = t1 - t0;
    ws.phase_cycles[6] = c_panel;
    ws.phase_cycles[7] = c_upd;
    ws.phase_cycles[1] = c_fn;
  }
  if (__syncthreads_or(bad) && tid == 0) {
    ws.fail = 1;
    atomicAdd(bv.error_count, 1);
  }
  // ---- 3. the factor and the row map to HBM for the dense kernel
  double* dst = bv.sn_lv + W.snlv_off;
  for (int e = tid; e < P.nLv; e += NT) dst[e] = Lv[e];
  for (int r = tid; r < n; r += NT) bv.sn_r2p[W.snr2p_off + r] = row2pos[r];
}

size_t snfactor_smem_bytes(int nLv, int S) {
  const size_t Sp = (size_t)pad2(S);
  return 8 * ((size_t)pad2(nLv) + Sp) + 2 * 2 * Sp;
}

cudaError_t launch_snfactor(const BatchView& bv, const StepParams& sp, const int32_t* worlds, int count, size_t smem,
                            cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  static SmemAttrCache attr;
  {
    const cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(snfactor_kernel), smem, attr);
    if (e != cudaSuccess) return e;
  }
  snfactor_kernel<<<count, kFactorThreads, smem, s>>>(bv, sp, worlds);
  return cudaGetLastError();
}

}  // namespace kd
