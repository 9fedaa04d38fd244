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
//   4. instruction streams: factor (scalar left-looking Cholesky entries plus
//      the inverse of every supernode's diagonal block), forward/backward solve
//      phases; each level packed onto 32 lanes.
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

// Longest-processing-time packing of one level's ops onto 32 lanes, laid out
// [step][lane]; returns the step count and the heaviest lane's cost.
template <class Op>
void pack_level(const std::vector<Op>& ops, const std::vector<int>& cost, const Op& nop, std::vector<Op>& out,
                int& steps, int& crit) {
  std::vector<int> idx(ops.size());
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return cost[a] > cost[b]; });
  std::vector<std::vector<int>> lanes(32);
  std::vector<int64_t> load(32, 0);
  for (int i : idx) {
    int l = 0;
    for (int k = 1; k < 32; ++k)
      if (load[k] < load[l]) l = k;
    lanes[l].push_back(i);
    load[l] += cost[i];
  }
  steps = 0;
  crit = 0;
  for (int l = 0; l < 32; ++l) {
    steps = std::max(steps, (int)lanes[l].size());
    crit = std::max<int>(crit, (int)load[l]);
  }
  for (int s = 0; s < steps; ++s)
    for (int l = 0; l < 32; ++l) out.push_back(s < (int)lanes[l].size() ? ops[lanes[l][s]] : nop);
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
  p.n_super = K;
  std::vector<int> snid(S);
  for (int k = 0; k < K; ++k)
    for (int j = sn_start[k]; j < sn_start[k + 1]; ++j) snid[j] = k;
  // row patterns
  std::vector<std::vector<int>> rp(S);
  for (int j = 0; j < S; ++j)
    for (int i : cs[j]) rp[i].push_back(j);
  // ---- Lv layout
  std::vector<int32_t> Lidx((size_t)S * S, -1), Xidx;
  std::vector<int> rpos(S);
  int nLv = 0;
  for (int j = 0; j < S; ++j) {
    rpos[j] = nLv++;
    for (int i : cs[j]) Lidx[(size_t)i * S + j] = nLv++;
  }
  p.nnzL = nLv;
  Xidx.assign((size_t)S * S, -1);
  for (int k = 0; k < K; ++k)
    for (int j = sn_start[k]; j < sn_start[k + 1]; ++j) {
      Xidx[(size_t)j * S + j] = rpos[j];
      for (int i = j + 1; i < sn_start[k + 1]; ++i) Xidx[(size_t)i * S + j] = nLv++;
    }
  if (nLv >= 65535) {
    why = "factor too large for 16-bit indices";
    return false;
  }
  p.nLv = nLv;
  {  // per-warp shared memory of kd_sparse.cu: Lv | v t | 8 PADMM vectors | 2 int16 maps
    const int Sp = (S + 1) & ~1;
    p.smem_doubles = ((nLv + 1) & ~1) + 10 * Sp + (Sp + 1) / 2 + 1;
  }
  auto L = [&](int i, int j) { return Lidx[(size_t)i * S + j]; };
  auto X = [&](int i, int j) { return Xidx[(size_t)i * S + j]; };
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
      g.dst = (uint16_t)(s == t ? rpos[ps] : L(std::max(ps, pt), std::min(ps, pt)));
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
  // ---- factor program, level-scheduled
  {
    std::vector<int> ready(nLv, 0);
    struct Pending {
      SnOp op;
      std::vector<uint32_t> terms;
    };
    std::vector<std::vector<Pending>> levels;
    auto add = [&](uint16_t kind, int dst, int aux, std::vector<uint32_t>&& terms) {
      int lv = ready[dst];
      if (kind == SN_OFF) lv = std::max(lv, ready[aux]);
      for (uint32_t t : terms) lv = std::max({lv, ready[t & 0xffff], ready[t >> 16]});
      ++lv;
      ready[dst] = lv;
      if ((int)levels.size() < lv) levels.resize(lv);
      p.factor_terms += (int64_t)terms.size();
      Pending pd;
      pd.op = SnOp{(uint16_t)dst, (uint16_t)aux, (uint16_t)terms.size(), kind, 0, 0};
      pd.terms = std::move(terms);
      levels[lv - 1].push_back(std::move(pd));
    };
    for (int j = 0; j < S; ++j) {
      std::vector<uint32_t> t;
      for (int k : rp[j]) t.push_back((uint32_t)L(j, k) | ((uint32_t)L(j, k) << 16));
      add(SN_DIAG, rpos[j], rpos[j], std::move(t));
      for (int i : cs[j]) {
        std::vector<uint32_t> u;
        size_t a = 0, b = 0;
        while (a < rp[i].size() && b < rp[j].size()) {  // common k < j, ascending
          if (rp[i][a] == rp[j][b]) {
            u.push_back((uint32_t)L(i, rp[i][a]) | ((uint32_t)L(j, rp[j][b]) << 16));
            ++a;
            ++b;
          } else if (rp[i][a] < rp[j][b]) {
            ++a;
          } else {
            ++b;
          }
        }
        add(SN_OFF, L(i, j), rpos[j], std::move(u));
      }
    }
    for (int k = 0; k < K; ++k)
      for (int j = sn_start[k]; j < sn_start[k + 1]; ++j)
        for (int i = j + 1; i < sn_start[k + 1]; ++i) {
          std::vector<uint32_t> t;
          for (int q = j; q < i; ++q) t.push_back((uint32_t)L(i, q) | ((uint32_t)X(q, j) << 16));
          add(SN_OFF, X(i, j), rpos[i], std::move(t));
        }
    const SnOp nop{0, 0, 0, SN_NOP, 0, 0};
    for (auto& lvl : levels) {
      std::vector<SnOp> ops;
      std::vector<int> cost;
      for (auto& pd : lvl) {
        SnOp o = pd.op;
        o.toff = (uint32_t)p.fterms.size();
        p.fterms.insert(p.fterms.end(), pd.terms.begin(), pd.terms.end());
        ops.push_back(o);
        cost.push_back(2 + (int)pd.terms.size());
      }
      SnPhase ph{(int32_t)p.fops.size(), 0, 0, 0};
      int crit = 0;
      pack_level(ops, cost, nop, p.fops, ph.steps, crit);
      p.factor_crit += crit;
      p.fphase.push_back(ph);
    }
  }
  // dense LLT of the capacity system, for the statistics
  p.dense_factor_terms = (int64_t)S * S * S / 6;
  // ---- solve program over supernode levels
  {
    std::vector<int> slev(K, 0);
    for (int k = 0; k < K; ++k)
      for (int j = sn_start[k]; j < sn_start[k + 1]; ++j)
        for (int i : cs[j])
          if (snid[i] != k) slev[snid[i]] = std::max(slev[snid[i]], slev[k] + 1);
    const int H = K ? *std::max_element(slev.begin(), slev.end()) + 1 : 0;
    p.s_levels = H;
    const SnSOp nop{0xffff, 0, 0};
    auto emit_phase = [&](int mode, std::vector<std::pair<int, std::vector<uint32_t>>>& rows) {
      std::vector<SnSOp> ops;
      std::vector<int> cost;
      for (auto& r : rows) {
        ops.push_back(SnSOp{(uint16_t)r.first, (uint16_t)r.second.size(), (uint32_t)p.sterms.size()});
        p.sterms.insert(p.sterms.end(), r.second.begin(), r.second.end());
        cost.push_back(2 + (int)r.second.size());
        p.solve_terms += (int64_t)r.second.size();
      }
      SnPhase ph{(int32_t)p.sops.size(), 0, mode, 0};
      int crit = 0;
      pack_level(ops, cost, nop, p.sops, ph.steps, crit);
      p.solve_crit += crit;
      p.sphase.push_back(ph);
    };
    auto term = [](int a, int v) { return (uint32_t)a | ((uint32_t)v << 16); };
    for (int lv = 0; lv < H; ++lv) {  // forward: L y = b
      std::vector<std::pair<int, std::vector<uint32_t>>> A_, B_;
      for (int k = 0; k < K; ++k) {
        if (slev[k] != lv) continue;
        const int c0 = sn_start[k], c1 = sn_start[k + 1];
        for (int i = c0; i < c1; ++i) {
          std::vector<uint32_t> t;
          for (int j : rp[i])
            if (j < c0) t.push_back(term(L(i, j), j));
          A_.push_back({i, std::move(t)});
          std::vector<uint32_t> u;
          for (int q = c0; q <= i; ++q) u.push_back(term(X(i, q), q));
          B_.push_back({i, std::move(u)});
        }
      }
      emit_phase(0, A_);
      emit_phase(1, B_);
    }
    for (int lv = H - 1; lv >= 0; --lv) {  // backward: L^T x = y
      std::vector<std::pair<int, std::vector<uint32_t>>> A_, B_;
      for (int k = 0; k < K; ++k) {
        if (slev[k] != lv) continue;
        const int c0 = sn_start[k], c1 = sn_start[k + 1];
        for (int j = c0; j < c1; ++j) {
          std::vector<uint32_t> t;
          for (int i : cs[j])
            if (i >= c1) t.push_back(term(L(i, j), i));
          A_.push_back({j, std::move(t)});
          std::vector<uint32_t> u;
          for (int q = j; q < c1; ++q) u.push_back(term(X(q, j), q));
          B_.push_back({j, std::move(u)});
        }
      }
      emit_phase(0, A_);
      emit_phase(1, B_);
    }
  }
  return true;
}

bool sn_plan_cpu_solve(const SnPlanHost& p, const double* D, const uint8_t* active, const double* b, double* x) {
  const int S = p.S;
  std::vector<double> Lv(p.nLv, 0.0), v(S, 0.0), t(S, 0.0);
  for (const SnGram& g : p.gram) {
    if (!active[g.s] || !active[g.t]) {
      if (g.flags & SG_DIAG) Lv[g.dst] = 1.0;
      continue;
    }
    Lv[g.dst] = D[(size_t)g.s * S + g.t];
  }
  bool ok = true;
  for (const SnPhase& ph : p.fphase)
    for (int k = 0; k < 32 * ph.steps; ++k) {
      const SnOp& o = p.fops[ph.off + k];
      if (o.kind == SN_NOP) continue;
      double acc = Lv[o.dst];
      for (int q = 0; q < o.nterm; ++q) {
        const uint32_t tt = p.fterms[o.toff + q];
        acc -= Lv[tt & 0xffff] * Lv[tt >> 16];
      }
      if (o.kind == SN_DIAG) {
        if (!(acc > 0.0)) ok = false;
        Lv[o.dst] = 1.0 / std::sqrt(acc);
      } else {
        Lv[o.dst] = acc * Lv[o.aux];
      }
    }
  for (int s = 0; s < S; ++s) v[p.slot_pos[s]] = active[s] ? b[s] : 0.0;
  for (const SnPhase& ph : p.sphase)
    for (int k = 0; k < 32 * ph.steps; ++k) {
      const SnSOp& o = p.sops[ph.off + k];
      if (o.dst == 0xffff) continue;
      if (ph.mode == 0) {
        double acc = v[o.dst];
        for (int q = 0; q < o.nterm; ++q) {
          const uint32_t tt = p.sterms[o.toff + q];
          acc -= Lv[tt & 0xffff] * v[tt >> 16];
        }
        t[o.dst] = acc;
      } else {
        double acc = 0.0;
        for (int q = 0; q < o.nterm; ++q) {
          const uint32_t tt = p.sterms[o.toff + q];
          acc += Lv[tt & 0xffff] * t[tt >> 16];
        }
        v[o.dst] = acc;
      }
    }
  for (int s = 0; s < S; ++s) x[s] = v[p.slot_pos[s]];
  return ok;
}

}  // namespace kd
