// kd_snplan.cpp — host construction of the supernodal sparse LLT plan
// (see kd_snplan.h) and a CPU interpreter used only by the self-test.
//
// Steps (all on the slot graph of one model, S = row capacity):
//   1. pattern: slots s, t couple iff their rows share a (non-world) body —
//      exactly the nonzeros assemble_dense can produce (delassus.cpp:74-95);
//   2. minimum-degree ordering (ties -> lowest slot), then an elimination-tree
//      postorder so fundamental supernodes are contiguous;
//   3. symbolic factor (column structures), fundamental supernodes, and the
//      supernode level of each block for the triangular solves;
//   4. per-world array layout (one dense panel per supernode + the inverse of
//      its diagonal block), the ancestor-update target maps of the panel
//      factor, and the chunked forward/backward solve program.
#include "kd_snplan.h"

#include <algorithm>
#include <cmath>
#include <numeric>

#include "kd_host.h"

namespace kd {

namespace {

struct BitMat {
  int n = 0, w = 0;
  std::vector<uint64_t> d;
  void init(int n_) {
    n = n_;
    w = (n + 63) / 64;
    d.assign((size_t)n * w, 0);
  }
  uint64_t* row(int i) { return d.data() + (size_t)i * w; }
  const uint64_t* row(int i) const { return d.data() + (size_t)i * w; }
  void set(int i, int j) { row(i)[j >> 6] |= 1ull << (j & 63); }
  bool get(int i, int j) const { return (row(i)[j >> 6] >> (j & 63)) & 1ull; }
};

// Column structures (positions > j) of the Cholesky factor of the pattern A.
void symbolic(const BitMat& A, std::vector<std::vector<int>>& cs) {
  BitMat G = A;
  const int n = A.n;
  cs.assign(n, {});
  for (int j = 0; j < n; ++j) {
    std::vector<int>& c = cs[j];
    for (int u = j + 1; u < n; ++u)
      if (G.get(j, u)) c.push_back(u);
    for (int x : c) {
      uint64_t* rx = G.row(x);
      for (int y : c)
        if (y != x) rx[y >> 6] |= 1ull << (y & 63);
    }
  }
}

}  // namespace

bool build_sn_plan(const HostModel& m, SnPlanHost& p, std::string& why) {
  p = SnPlanHost{};
  p.n_jd = m.n_bil + m.n_dyn;
  p.lim_base = p.n_jd;
  // Planned slots: every static row, both bounds of every limited joint, and
  // the contact slots of body-world pairs.  Body-body pairs (e.g. two sphere
  // pads of one foot) would couple otherwise independent subtrees of the
  // elimination order for contacts that almost never exist; they are left out,
  // and a world that activates one takes the dense kernel for that step.
  int S = p.lim_base + 2 * m.info.n_limited_joints;
  int body_body = 0;
  for (const DevPair& pr : m.pairs) body_body += m.geoms[pr.a].body >= 0 && m.geoms[pr.b].body >= 0;
  if (body_body > (int)m.bodies.size()) {  // contact-dominated scenes (piles): no static structure to exploit
    why = std::to_string(body_body) + " body-body collision pairs";
    return false;
  }
  for (const DevPair& pr : m.pairs) {
    const bool world = m.geoms[pr.a].body < 0 || m.geoms[pr.b].body < 0;
    p.pair_slot.push_back(world ? S : -1);
    if (world) S += 3 * (pr.kind == P_BOX_PLANE ? 4 : 1);
  }
  p.S = S;
  if (S <= 0) {
    why = "no rows";
    return false;
  }
  if (S > 2048) {
    why = "planned slots " + std::to_string(S) + " > 2048";
    return false;
  }
  // ---- slot bodies (the row layout of model.cpp:254-276 + K1's limit/contact slots)
  std::vector<int32_t>& sb = p.slot_body;
  sb.assign(2 * S, -1);
  for (const DevJoint& j : m.joints) {
    for (int r = 0; r < j.row_count; ++r) {
      sb[2 * (j.row_offset + r)] = j.child;
      sb[2 * (j.row_offset + r) + 1] = j.parent;
    }
    const int nd = ((j.flags & JF_PD) ? 1 : 0) + ((j.flags & JF_ARMATURE) ? 1 : 0) + ((j.flags & JF_DAMPING) ? 1 : 0);
    for (int r = 0; r < nd; ++r) {
      sb[2 * (m.n_bil + j.dyn_offset + r)] = j.child;
      sb[2 * (m.n_bil + j.dyn_offset + r) + 1] = j.parent;
    }
    if (j.flags & JF_LIMITS)
      for (int bound = 0; bound < 2; ++bound) {
        sb[2 * (p.lim_base + 2 * j.limit_slot + bound)] = j.child;
        sb[2 * (p.lim_base + 2 * j.limit_slot + bound) + 1] = j.parent;
      }
  }
  for (size_t pi = 0; pi < m.pairs.size(); ++pi) {
    const DevPair& pr = m.pairs[pi];
    if (p.pair_slot[pi] < 0) continue;
    const int cap = pr.kind == P_BOX_PLANE ? 4 : 1;
    const int ba = m.geoms[pr.a].body, bb = m.geoms[pr.b].body;
    for (int k = 0; k < 3 * cap; ++k) {
      sb[2 * (p.pair_slot[pi] + k)] = ba;
      sb[2 * (p.pair_slot[pi] + k) + 1] = bb >= 0 ? bb : -1;
    }
  }
  auto shares = [&](int s, int t) {
    for (int u = 0; u < 2; ++u)
      for (int v = 0; v < 2; ++v)
        if (sb[2 * s + u] >= 0 && sb[2 * s + u] == sb[2 * t + v]) return true;
    return false;
  };
  // ---- pattern and minimum-degree ordering
  BitMat A;
  A.init(S);
  for (int s = 0; s < S; ++s)
    for (int t = 0; t < s; ++t)
      if (shares(s, t)) {
        A.set(s, t);
        A.set(t, s);
      }
  std::vector<int> order;
  {
    BitMat G = A;
    std::vector<uint64_t> alive(A.w, 0);
    for (int v = 0; v < S; ++v) alive[v >> 6] |= 1ull << (v & 63);
    for (int it = 0; it < S; ++it) {
      int best = -1, bdeg = 1 << 30;
      for (int v = 0; v < S; ++v) {
        if (!((alive[v >> 6] >> (v & 63)) & 1)) continue;
        int deg = 0;
        const uint64_t* r = G.row(v);
        for (int k = 0; k < A.w; ++k) deg += __builtin_popcountll(r[k] & alive[k]);
        if (deg < bdeg) {
          bdeg = deg;
          best = v;
        }
      }
      order.push_back(best);
      alive[best >> 6] &= ~(1ull << (best & 63));
      std::vector<int> nb;
      for (int u = 0; u < S; ++u)
        if (((alive[u >> 6] >> (u & 63)) & 1) && G.get(best, u)) nb.push_back(u);
      for (int x : nb) {
        uint64_t* rx = G.row(x);
        for (int y : nb)
          if (y != x) rx[y >> 6] |= 1ull << (y & 63);
      }
    }
  }
  auto permuted = [&](const std::vector<int>& ord, BitMat& P) {
    std::vector<int> pos(S);
    for (int k = 0; k < S; ++k) pos[ord[k]] = k;
    P.init(S);
    for (int s = 0; s < S; ++s)
      for (int t = 0; t < S; ++t)
        if (A.get(s, t)) P.set(pos[s], pos[t]);
  };
  std::vector<std::vector<int>> cs;
  {
    BitMat P;
    permuted(order, P);
    symbolic(P, cs);
    // elimination-tree postorder (children ascending)
    std::vector<std::vector<int>> ch(S);
    std::vector<int> roots;
    for (int j = 0; j < S; ++j) {
      if (cs[j].empty()) roots.push_back(j);
      else ch[cs[j][0]].push_back(j);
    }
    std::vector<int> post;
    for (int r : roots) {
      std::vector<std::pair<int, int>> st{{r, 0}};
      while (!st.empty()) {
        auto& top = st.back();
        if (top.second < (int)ch[top.first].size()) {
          const int c = ch[top.first][top.second++];
          st.push_back({c, 0});
        } else {
          post.push_back(top.first);
          st.pop_back();
        }
      }
    }
    std::vector<int> o2(S);
    for (int k = 0; k < S; ++k) o2[k] = order[post[k]];
    order = o2;
    permuted(order, P);
    symbolic(P, cs);
  }
  p.slot_pos.resize(S);
  for (int k = 0; k < S; ++k) p.slot_pos[order[k]] = (uint16_t)k;
  // ---- fundamental supernodes
  std::vector<int> nchild(S, 0);
  for (int j = 0; j < S; ++j)
    if (!cs[j].empty()) ++nchild[cs[j][0]];
  std::vector<int> sn_start{0};
  for (int j = 1; j < S; ++j) {
    const int q = j - 1;
    const bool merge = !cs[q].empty() && cs[q][0] == j && nchild[j] == 1 && cs[q].size() == cs[j].size() + 1 &&
                       j - sn_start.back() < 32;
    if (!merge) sn_start.push_back(j);
  }
  sn_start.push_back(S);
  const int K = (int)sn_start.size() - 1;
  std::vector<int> snid(S);
  for (int k = 0; k < K; ++k)
    for (int j = sn_start[k]; j < sn_start[k + 1]; ++j) snid[j] = k;
  // nonzero tiles of L (the hand-off's L^-1 skips the zero ones)
  if (S <= 256) {
    p.lmask = 0;
    for (int j = 0; j < S; ++j) {
      p.lmask |= 1ull << ((j / 32) * (j / 32 + 1) / 2 + j / 32);
      for (int i : cs[j]) p.lmask |= 1ull << ((i / 32) * (i / 32 + 1) / 2 + j / 32);
    }
    // column groups (4 wide, the DMMA k step) of every L tile that hold a
    // nonzero: the L^-1 tile products skip the others (their terms are exact zeros)
    p.kmask.assign(36, 0);
    for (int j = 0; j < S; ++j) {
      p.kmask[(j / 32) * (j / 32 + 1) / 2 + j / 32] |= (uint8_t)(1u << ((j % 32) / 4));
      for (int i : cs[j]) p.kmask[(i / 32) * (i / 32 + 1) / 2 + j / 32] |= (uint8_t)(1u << ((j % 32) / 4));
    }
    // X = L^-1: X_ij != 0 only if i is j or an elimination-tree ancestor of j
    p.xmask = 0;
    for (int j = 0; j < S; ++j)
      for (int i = j;; i = cs[i][0]) {
        p.xmask |= 1ull << ((i / 32) * (i / 32 + 1) / 2 + j / 32);
        if (cs[i].empty()) break;
      }
  } else {
    p.lmask = p.xmask = ~0ull;
    p.kmask.assign(36, 0xff);
  }
  // row patterns
  std::vector<std::vector<int>> rp(S);
  for (int j = 0; j < S; ++j)
    for (int i : cs[j]) rp[i].push_back(j);
  // ---- Lv layout: one dense panel per supernode, then the X blocks
  std::vector<int32_t> Lidx((size_t)S * S, -1);
  int nLv = 0;
  p.sup.resize(K);
  std::vector<int> qpos(S, -1);
  for (int k = 0; k < K; ++k) {
    SnSuper& u = p.sup[k];
    const int c0 = sn_start[k], c1 = sn_start[k + 1];
    std::vector<int> R;
    for (int i : cs[c1 - 1]) R.push_back(i);
    u.c0 = c0;
    u.w = c1 - c0;
    u.m = (int)R.size();
    u.ld = (u.w + u.m) | 1;
    u.pb = nLv;
    nLv += u.ld * u.w;
    u.prow_off = (int)p.prow.size();
    for (int q = 0; q < u.w; ++q) p.prow.push_back(c0 + q);
    p.prow.insert(p.prow.end(), R.begin(), R.end());
    if (u.m > 255 || u.w > 32) {
      why = "supernode too large";
      return false;
    }
    for (int q = 0; q < u.w; ++q) qpos[c0 + q] = q;
    for (int q = 0; q < u.m; ++q) qpos[R[q]] = u.w + q;
    for (int j = c0; j < c1; ++j) {
      Lidx[(size_t)j * S + j] = u.pb + (j - c0) * u.ld + (j - c0);
      for (int i : cs[j]) Lidx[(size_t)i * S + j] = u.pb + (j - c0) * u.ld + qpos[i];
    }
    for (int q = 0; q < u.w; ++q) qpos[c0 + q] = -1;
    for (int q = 0; q < u.m; ++q) qpos[R[q]] = -1;
    p.nnzL += u.w * (u.w + 1) / 2 + u.w * u.m;
  }
  for (int k = 0; k < K; ++k) {  // X = L_SS^-1 lives (transposed) in the panel's unused upper triangle
    SnSuper& u = p.sup[k];
    u.ws = u.ld;
    u.xb = u.pb;
  }
  if (nLv >= 65535) {
    why = "factor too large for 16-bit indices";
    return false;
  }
  p.nLv = nLv;
  auto L = [&](int i, int j) { return Lidx[(size_t)i * S + j]; };
  auto X = [&](int i, int j) {  // i >= j, same supernode
    const SnSuper& u = p.sup[snid[j]];
    return u.xb + (i - u.c0) * u.ws + (j - u.c0);
  };
  // ---- hand-off scatter list: panel (lower) entries -> kd_dense.cu's tile
  // layout for n = S (tiles of 32, off-diagonal row stride 33, packed
  // diagonal tiles)
  {
    auto rows_of = [&](int ti) { return std::min(32, S - 32 * ti); };
    auto lidx = [&](int i, int j) {
      const int ti = i >> 5, tj = j >> 5, r = i & 31, c = j & 31;
      const int base = 528 * ti * ti;
      if (ti == tj) return base + ti * 33 * rows_of(ti) + ((r * (r + 1)) >> 1) + c;
      return base + tj * 33 * rows_of(ti) + r * 33 + c;
    };
    for (const SnSuper& u : p.sup)
      for (int c = 0; c < u.w; ++c)
        for (int q = c; q < u.w + u.m; ++q) {
          const int li = lidx(p.prow[u.prow_off + q], u.c0 + c);
          if (li >= 65536) {
            p.scat.clear();
            break;
          }
          p.scat.push_back((uint32_t)(u.pb + c * u.ld + q) | ((uint32_t)li << 16));
        }
  }
  // ---- ancestor-update target maps
  for (int k = 0; k < K; ++k) {
    SnSuper& u = p.sup[k];
    u.tmap_off = (int)p.tmap.size();
    const int c1 = u.c0 + u.w;
    const std::vector<int>& R = cs[c1 - 1];
    for (int ri = 0; ri < u.m; ++ri)
      for (int rj = 0; rj <= ri; ++rj) {
        const int idx = L(R[ri], R[rj]);
        if (idx < 0) {
          why = "symbolic factor inconsistent";
          return false;
        }
        p.tmap.push_back((uint32_t)idx | ((uint32_t)ri << 16) | ((uint32_t)rj << 24));
      }
    p.factor_fma += (int64_t)u.m * (u.m + 1) / 2 * u.w + (int64_t)(u.w + u.m) * u.w * u.w / 2;
  }
  p.dense_factor_fma = (int64_t)S * S * S / 6;
  // ---- Gram entries (slot order, s >= t)
  for (int s = 0; s < S; ++s)
    for (int t = 0; t <= s; ++t) {
      if (s != t && !shares(s, t)) continue;
      int bodies[2], ns = 0;
      for (int u = 0; u < 2; ++u) {
        const int b = sb[2 * s + u];
        if (b < 0) continue;
        if (sb[2 * t] == b || sb[2 * t + 1] == b) bodies[ns++] = b;
      }
      if (ns == 2 && bodies[1] < bodies[0]) std::swap(bodies[0], bodies[1]);
      if (ns == 0) continue;
      SnGram g{};
      const int ps = p.slot_pos[s], pt = p.slot_pos[t];
      g.dst = (uint16_t)L(std::max(ps, pt), std::min(ps, pt));
      g.s = (uint16_t)s;
      g.t = (uint16_t)t;
      uint16_t f = s == t ? SG_DIAG : 0;
      if (sb[2 * s] != bodies[0]) f |= SG_S1;
      if (sb[2 * t] != bodies[0]) f |= SG_T1;
      if (ns == 2) {
        f |= SG_TWO;
        if (sb[2 * s] != bodies[1]) f |= SG_S2;
        if (sb[2 * t] != bodies[1]) f |= SG_T2;
      }
      g.flags = f;
      p.gram.push_back(g);
    }
  // ---- per-body Gram lists: bodies ascending; a body's rows in slot order.
  // An entry shared by two bodies b1 < b2 is stored by b1 and accumulated by
  // b2, which is assemble_dense's ascending body order (delassus.cpp:80-95).
  {
    const int nbod = (int)m.bodies.size();
    std::vector<std::vector<uint32_t>> bsl(nbod);
    std::vector<std::vector<int>> local(nbod, std::vector<int>(S, -1));
    for (int sl = 0; sl < S; ++sl)
      for (int u = 0; u < 2; ++u) {
        const int b = sb[2 * sl + u];
        if (b < 0) continue;
        local[b][sl] = (int)bsl[b].size();
        bsl[b].push_back((uint32_t)sl | ((uint32_t)u << 16));
      }
    std::vector<std::vector<uint32_t>> st(nbod), ac(nbod);
    int kmax = 0;
    for (int b = 0; b < nbod; ++b) kmax = std::max(kmax, (int)bsl[b].size());
    const int Sp = (S + 1) & ~1;
    if (kmax > 255) {
      why = "a body carries too many rows for the staged Gram";
      return false;
    }
    p.kmax = kmax;
    p.vreg = std::max(7 * Sp, 12 * kmax + Sp);  // PADMM vectors, or Gram staging + P
    for (const SnGram& g : p.gram) {
      int bodies[2], ns = 0;
      for (int u = 0; u < 2; ++u) {
        const int b = sb[2 * g.s + u];
        if (b >= 0 && (sb[2 * g.t] == b || sb[2 * g.t + 1] == b)) bodies[ns++] = b;
      }
      if (ns == 2 && bodies[1] < bodies[0]) std::swap(bodies[0], bodies[1]);
      for (int k = 0; k < ns; ++k) {
        const int b = bodies[k];
        const uint32_t word = (uint32_t)g.dst | ((uint32_t)local[b][g.s] << 16) | ((uint32_t)local[b][g.t] << 24);
        (k == 0 ? st[b] : ac[b]).push_back(word);
      }
    }
    for (int b = 0; b < nbod; ++b) {
      SnGBody gb{};
      gb.slot_off = (int)p.gslot.size();
      gb.k = (int)bsl[b].size();
      p.gslot.insert(p.gslot.end(), bsl[b].begin(), bsl[b].end());
      gb.pair_off = (int)p.gpair.size();
      gb.n_store = (int)st[b].size();
      gb.n_acc = (int)ac[b].size();
      p.gpair.insert(p.gpair.end(), st[b].begin(), st[b].end());
      p.gpair.insert(p.gpair.end(), ac[b].begin(), ac[b].end());
      p.gbody.push_back(gb);
    }
  }
  // ---- solve program over supernode levels
  std::vector<int> slev(K, 0);
  for (int k = 0; k < K; ++k)
    for (int j = sn_start[k]; j < sn_start[k + 1]; ++j)
      for (int i : cs[j])
        if (snid[i] != k) slev[snid[i]] = std::max(slev[snid[i]], slev[k] + 1);
  const int H = K ? *std::max_element(slev.begin(), slev.end()) + 1 : 0;
  p.s_levels = H;
  struct Row {
    int dst;
    std::vector<uint32_t> terms;
  };
  struct PhaseBuild {
    int mode;
    std::vector<Row> rows;
  };
  std::vector<PhaseBuild> phases;
  auto term = [](int a, int v) { return (uint32_t)a | ((uint32_t)v << 16); };
  for (int lv = 0; lv < H; ++lv) {  // forward: L y = b
    PhaseBuild A{0, {}}, B{1, {}};
    for (int k = 0; k < K; ++k) {
      if (slev[k] != lv) continue;
      const int c0 = sn_start[k], c1 = sn_start[k + 1];
      for (int i = c0; i < c1; ++i) {
        Row a{i, {}}, b{i, {}};
        for (int j : rp[i])
          if (j < c0) a.terms.push_back(term(L(i, j), j));
        for (int q = c0; q <= i; ++q) b.terms.push_back(term(X(i, q), q));
        A.rows.push_back(std::move(a));
        B.rows.push_back(std::move(b));
      }
    }
    phases.push_back(std::move(A));
    phases.push_back(std::move(B));
  }
  for (int lv = H - 1; lv >= 0; --lv) {  // backward: L^T x = y
    PhaseBuild A{0, {}}, B{1, {}};
    for (int k = 0; k < K; ++k) {
      if (slev[k] != lv) continue;
      const int c0 = sn_start[k], c1 = sn_start[k + 1];
      for (int j = c0; j < c1; ++j) {
        Row a{j, {}}, b{j, {}};
        for (int i : cs[j])
          if (i >= c1) a.terms.push_back(term(L(i, j), i));
        for (int q = j; q < c1; ++q) b.terms.push_back(term(X(q, j), q));
        A.rows.push_back(std::move(a));
        B.rows.push_back(std::move(b));
      }
    }
    phases.push_back(std::move(A));
    phases.push_back(std::move(B));
  }
  // blob: phase table, then records, then terms
  std::vector<uint32_t>& blob = p.prog;
  const int nph = (int)phases.size();
  p.n_sph = nph;
  blob.assign(4 * nph, 0);
  std::vector<uint32_t> terms_all;
  struct Rec {
    uint32_t w0, toff, flags;
  };
  std::vector<std::vector<Rec>> recs(nph);
  std::vector<std::vector<std::vector<uint32_t>>> rec_terms(nph);
  for (int ph = 0; ph < nph; ++ph) {
    const PhaseBuild& P = phases[ph];
    int maxn = 1;
    for (const Row& r : P.rows) maxn = std::max(maxn, (int)r.terms.size());
    // chunk size (<= kSnChunk, the device's unrolled width): minimise a
    // latency estimate — each step costs about two dependent shared-memory
    // round trips plus the chunk's FMA chain, a split phase one more pass
    int bestC = 1, bestSlots = 0;
    double bestCost = 1e30;
    for (int C = 1; C <= std::min(maxn, kSnChunk); ++C) {
      int slots = 0;
      bool split = false;
      for (const Row& r : P.rows) {
        const int ch = std::max(1, ((int)r.terms.size() + C - 1) / C);
        slots += ch;
        split |= ch > 1;
      }
      const int steps = (slots + 31) / 32;
      const double cost = steps * (100.0 + 3.0 * C) + (split ? 90.0 : 0.0);
      if (cost < bestCost || (cost == bestCost && C > bestC)) {
        bestCost = cost;
        bestC = C;
        bestSlots = slots;
      }
    }
    const int C = bestC;
    const int steps = (bestSlots + 31) / 32;
    bool split = false;
    int crit = 0;
    std::vector<int> lane_load(32, 0);
    recs[ph].assign(32 * std::max(steps, 0), Rec{0, 0, 0});
    rec_terms[ph].assign(recs[ph].size(), {});
    int slot = 0;
    for (const Row& r : P.rows) {
      const int n = (int)r.terms.size();
      const int ch = std::max(1, (n + C - 1) / C);
      split |= ch > 1;
      for (int c = 0; c < ch; ++c) {
        const int b0 = c * C, b1 = std::min(n, b0 + C);
        Rec& rc = recs[ph][slot];
        rc.w0 = (uint32_t)r.dst | ((uint32_t)(b1 - b0) << 16);
        rc.flags = (1u << 31) | (c == 0 ? (1u << 30) | ((uint32_t)(ch - 1) << 24) : 0u);
        rec_terms[ph][slot].assign(r.terms.begin() + b0, r.terms.begin() + b1);
        lane_load[slot & 31] += b1 - b0;
        p.solve_terms += b1 - b0;
        ++slot;
      }
    }
    for (int l = 0; l < 32; ++l) crit = std::max(crit, lane_load[l]);
    p.solve_crit += crit;
    p.max_slots = std::max(p.max_slots, 32 * steps);
    blob[4 * ph + 1] = (uint32_t)steps;
    blob[4 * ph + 2] = (uint32_t)P.mode;
    blob[4 * ph + 3] = split ? 1u : 0u;
  }
  for (int ph = 0; ph < nph; ++ph) {  // records (8-byte aligned)
    if (blob.size() & 1) blob.push_back(0);
    blob[4 * ph] = (uint32_t)blob.size();
    for (size_t r = 0; r < recs[ph].size(); ++r) {
      blob.push_back(recs[ph][r].w0);
      blob.push_back(0);  // patched with the term offset below
    }
  }
  for (int ph = 0; ph < nph; ++ph)
    for (size_t r = 0; r < recs[ph].size(); ++r) {
      const uint32_t toff = (uint32_t)blob.size();
      blob.insert(blob.end(), rec_terms[ph][r].begin(), rec_terms[ph][r].end());
      if (toff >= (1u << 24)) {
        why = "solve program too large";
        return false;
      }
      blob[blob[4 * ph] + 2 * r + 1] = toff | recs[ph][r].flags;
    }
  {  // per-warp shared memory of kd_sparse.cu: Lv | v t + 5 PADMM vectors (or Gram staging) | partials | 2 int16 maps
    const int Sp = (S + 1) & ~1;
    p.smem_doubles = ((nLv + 1) & ~1) + p.vreg + p.max_slots + (Sp + 1) / 2 + 1;
  }
  return true;
}

namespace {

// The device algorithms of kd_sparse.cu on the host (self-test).
bool cpu_factor(const SnPlanHost& p, std::vector<double>& Lv) {
  bool ok = true;
  for (const SnSuper& u : p.sup) {
    double* P = Lv.data() + u.pb;
    double* X = Lv.data() + u.xb;
    for (int c = 0; c < u.w; ++c) {
      const double d = P[c * u.ld + c];
      if (!(d > 0.0)) ok = false;
      const double r = 1.0 / std::sqrt(d);
      for (int q = c + 1; q < u.w + u.m; ++q) P[c * u.ld + q] *= r;
      X[c * u.ws + c] = r;  // the diagonal keeps 1/L_cc (L_cc itself is never read again)
      for (int q = c + 1; q < u.w + u.m; ++q) {
        const double lq = P[c * u.ld + q];
        for (int j = c + 1; j <= std::min(q, u.w - 1); ++j) P[j * u.ld + q] -= lq * P[c * u.ld + j];
      }
    }
    for (int j = 0; j < u.w; ++j)
      for (int i = j + 1; i < u.w; ++i) {
        double s = 0.0;
        for (int q = j; q < i; ++q) s += P[q * u.ld + i] * X[q * u.ws + j];
        X[i * u.ws + j] = -s * X[i * u.ws + i];
      }
    const int T = u.m * (u.m + 1) / 2;
    for (int e = 0; e < T; ++e) {
      const uint32_t te = p.tmap[u.tmap_off + e];
      const int ri = (te >> 16) & 0xff, rj = te >> 24;
      double s = 0.0;
      for (int c = 0; c < u.w; ++c) s += P[c * u.ld + u.w + ri] * P[c * u.ld + u.w + rj];
      Lv[te & 0xffff] -= s;
    }
  }
  return ok;
}

void cpu_solve(const SnPlanHost& p, const std::vector<double>& Lv, std::vector<double>& v) {
  const uint32_t* blob = p.prog.data();
  std::vector<double> t(p.S, 0.0), part(std::max(1, p.max_slots), 0.0);
  for (int ph = 0; ph < p.n_sph; ++ph) {
    const uint32_t rec0 = blob[4 * ph], steps = blob[4 * ph + 1], mode = blob[4 * ph + 2];
    auto finalize = [&](int dst, double s) {
      if (mode == 0) t[dst] = v[dst] - s;
      else v[dst] = s;
    };
    for (uint32_t slot = 0; slot < 32 * steps; ++slot) {
      const uint32_t w0 = blob[rec0 + 2 * slot], w1 = blob[rec0 + 2 * slot + 1];
      if (!(w1 >> 31)) continue;
      const int dst = w0 & 0xffff, nt = w0 >> 16;
      const uint32_t toff = w1 & 0xffffff;
      double pr[kSnChunk] = {};
      for (int k = 0; k < nt; ++k) {
        const uint32_t tt = blob[toff + k];
        pr[k] = Lv[tt & 0xffff] * (mode == 0 ? v : t)[tt >> 16];
      }
      const double s = ((pr[0] + pr[1]) + (pr[2] + pr[3])) + ((pr[4] + pr[5]) + (pr[6] + pr[7]));
      const bool owner = (w1 >> 30) & 1;
      const int npart = (w1 >> 24) & 63;
      if (owner && npart == 0) finalize(dst, s);
      else part[slot] = s;
    }
    for (uint32_t slot = 0; slot < 32 * steps; ++slot) {
      const uint32_t w0 = blob[rec0 + 2 * slot], w1 = blob[rec0 + 2 * slot + 1];
      const int npart = (w1 >> 24) & 63;
      if (!(w1 >> 31) || !((w1 >> 30) & 1) || npart == 0) continue;
      double s = part[slot];
      for (int q = 1; q <= npart; ++q) s += part[slot + q];
      finalize(w0 & 0xffff, s);
    }
  }
}

}  // namespace

bool sn_plan_cpu_solve(const SnPlanHost& p, const double* D, const uint8_t* active, const double* b, double* x) {
  const int S = p.S;
  std::vector<double> Lv(p.nLv, 0.0), v(S, 0.0);
  for (const SnGram& g : p.gram) {
    if (!active[g.s] || !active[g.t]) {
      if (g.flags & SG_DIAG) Lv[g.dst] = 1.0;
      continue;
    }
    Lv[g.dst] = D[(size_t)g.s * S + g.t];
  }
  const bool ok = cpu_factor(p, Lv);
  for (int s = 0; s < S; ++s) v[p.slot_pos[s]] = active[s] ? b[s] : 0.0;
  cpu_solve(p, Lv, v);
  for (int s = 0; s < S; ++s) x[s] = v[p.slot_pos[s]];
  return ok;
}

}  // namespace kd
