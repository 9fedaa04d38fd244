// kd_capi.cu — the C-ABI (include/kamino_b200.h): models, device-resident
// world batches, stepping and introspection.
//
// kd_batch is the device-side WorldBatch (batch.hpp:14-54).  Creation lays out
// every per-world slab (state, rows, bodies, contacts, caches) by prefix sums
// over model capacities, bins worlds by dense-Delassus shared-memory class, and
// uploads the immutable model tables once.  kd_batch_step runs, per step,
//   K1 assemble (warp/world) -> K2 dense (CTA/world, per bin)
//   -> K2g dense-global -> K2b matrix-free CR -> K3 recover (warp/world)
// on one stream; a K2 CTA exits immediately when its world chose another
// backend this step (the choice depends on the contact/limit count, known only
// on the device).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <type_traits>
#include <vector>

#include "kd_host.h"

using namespace kd;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define KD_CK(x)                                                                             \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess) return fail(KD_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct DevMem {
  std::vector<void*> ptrs;
  ~DevMem() {
    for (void* p : ptrs) cudaFree(p);
  }
  template <class T>
  cudaError_t alloc(T*& out, size_t count) {
    void* p = nullptr;
    const cudaError_t e = cudaMalloc(&p, std::max<size_t>(1, count) * sizeof(T));
    if (e == cudaSuccess) {
      // zero-fill on the legacy stream and wait for it: the batch streams are
      // non-blocking, so nothing else would order this fill before their work
      cudaMemset(p, 0, std::max<size_t>(1, count) * sizeof(T));
      cudaStreamSynchronize(0);
      ptrs.push_back(p);
      out = static_cast<T*>(p);
    }
    return e;
  }
  void release(void* p) {
    for (void*& q : ptrs)
      if (q == p) {
        cudaFree(q);
        q = nullptr;
      }
  }
};

// Per-world dense-global slab: the factor (tile layout) followed by the PADMM
// unit state y, z, y_hat, z_hat (4 x 32 T doubles) of dense_kernel<., true>.
int64_t slab_doubles(int cap) {
  const int64_t t = (cap + 31) / 32;
  return (((int64_t)dense_factor_doubles(cap) + 1) & ~(int64_t)1) + 4 * 32 * t + 2;
}

struct Bin {
  int cap = 0;  // rows (dense) / rows (cr)
  int nbcap = 0;
  int nt = 0;
  int count = 0;
  int32_t* d_worlds = nullptr;
  std::vector<int32_t> worlds;
  // every world's model is planned with all collision pairs in planned slots,
  // so K1 never sends one of them here (kd_assemble.cu backend choice): the
  // launch is skipped (an empty 1-CTA-per-world launch still costs ~10 us)
  bool never = false;
  bool rare = false;  // every world's model is planned: a world lands here only as a fallback
  // the batch's parts (world ranges [cut[p], cut[p+1])): this bin's worlds in each
  int hoff[4] = {0, 0, 0, 0}, hcount[4] = {0, 0, 0, 0};
  void set_parts(const int* cut, int np) {
    int k = 0;
    for (int p = 0; p < np; ++p) {
      hoff[p] = k;
      while (k < (int)worlds.size() && worlds[k] < cut[p + 1]) ++k;
      hcount[p] = k - hoff[p];
    }
  }
};

// dense shared-memory classes: (row capacity, threads per CTA)
constexpr int kClasses[4][2] = {{32, 64}, {64, 64}, {128, 128}, {232, 256}};
constexpr int kSmemMaxRows = 232;
constexpr int kDenseGlobalMaxRows = KD_DENSE_ROW_CROSSOVER;
constexpr size_t kSnMaxSmem = 232448;  // per-CTA shared memory opt-in limit (227 KB)
constexpr int kSnAutoMaxSlots = 32;     // supernodal kernel by default up to one dense tile
constexpr size_t kClPerCta = 233472 / 2;  // K2c: two CTAs per SM (228 KB of shared memory, 1 KB reserved per CTA)

}  // namespace

int kd::set_last_error(int code, const std::string& msg) { return fail(code, msg); }

struct kd_batch;
namespace {
cudaError_t to_dev(kd_batch* b, void* dst, const void* src, size_t bytes);
cudaError_t to_host(kd_batch* b, void* dst, const void* src, size_t bytes);
}  // namespace

struct kd_batch {
  int device = 0;
  cudaStream_t stream = nullptr;
  // large batches step as independent parts (contiguous world ranges) on
  // their own streams, so one part's kernel tails overlap the other parts'
  // kernels; KD_SPLIT=n sets the part count (1 disables, default 2)
  int n_halves = 1;
  int cut[5] = {0, 0, 0, 0, 0};
  cudaStream_t pstream[4] = {};
  cudaEvent_t ev_fork = nullptr, ev_join[4] = {};
  std::vector<HostModel> models;
  std::vector<int32_t> world_model;
  int n_worlds = 0;
  std::vector<DevWorld> worlds;
  std::vector<int32_t> pose_off, twist_off;
  std::vector<int64_t> row_off;
  int64_t total_rows = 0, pose_len = 0, twist_len = 0, total_lslab = 0;
  // the dense-global slab holds min(capacity, 300) rows per world (Auto never
  // factors more); the first step with backend = Dense re-sizes it to the full
  // row capacity of every world above 300 rows (build_backend factors densely
  // at any n, delassus.cpp:203-216)
  bool dense_full = false, has_big = false;
  int total_bodies = 0, total_contacts = 0, total_jcache = 0, total_lslots = 0;
  DevMem mem;
  BatchView view{};
  std::vector<Bin> dense_bins;
  Bin global_bin, cr_auto_bin, cr_all_bin;
  // supernodal sparse-LLT bins: one per planned model (worlds of one model per CTA)
  struct SnBin {
    int model = 0, per_warp = 0, wpc = 1, prog_words = 0;
    bool hand = false;  // hand-off model: K2f (factor only, CTA per world)
    size_t hand_smem = 0;
    Bin bin;
  };
  std::vector<SnBin> sn_bins;
  bool sparse = true;
  bool no_df = false;
  bool no_tmem = false;
  bool slab_sweep_forced = false;
  int sparse_mode = 1;
  bool sn_handoff = true;
  int64_t total_snlv = 0, total_snr2p = 0;
  // K2c (kd_dense_cl.cu, opt-in KD_CLUSTER=1): hand-off models whose X splits
  // over a CTA pair with two pairs' CTAs per SM (measured slower than K2 on
  // DR-Legs: DESIGN.md §7)
  bool cluster = false;
  std::vector<int> cl_split, cl_xlen;
  int64_t total_xslab = 0;
  size_t cl_smem = 0;
  int hist_cap = 0;
  double* d_hist = nullptr;
  double* d_nest = nullptr;  // Nesterov beta table (StepParams::nest_beta)
  int nest_cap = 0;
  int32_t* d_err = nullptr;
  bool timing = false;
  cudaEvent_t ev[6] = {};
  // per-step family events recorded without synchronising: resolved lazily
  // (kd_batch_get_timing / kd_batch_sync), so timing can stay on inside a
  // timed region without perturbing it
  std::vector<cudaEvent_t> evpool;  // 5 per step
  size_t ev_used = 0, ev_done = 0;
  double ms[4] = {0, 0, 0, 0};
  int64_t launches = 0;
  // one step captured as a CUDA graph and replayed for multi-step calls
  // (launch-bound small batches); re-captured when the step parameters or
  // the batch view change
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  StepParams graph_sp{};
  int graph_backend = -1, graph_launches = 0;
  bool graphs = true;
  void drop_graph() {
    if (graph_exec) cudaGraphExecDestroy(graph_exec);
    if (graph) cudaGraphDestroy(graph);
    graph_exec = nullptr;
    graph = nullptr;
  }
  ~kd_batch() {
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : evpool) cudaEventDestroy(e);
    drop_graph();
    if (ev_fork) cudaEventDestroy(ev_fork);
    for (int p = 1; p < 4; ++p) {
      if (ev_join[p]) cudaEventDestroy(ev_join[p]);
      if (pstream[p]) cudaStreamDestroy(pstream[p]);
    }
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {
// Host<->device copies of the batch API, ordered on the batch stream (which is
// non-blocking, so legacy-stream cudaMemcpy would race with in-flight steps):
// enqueue after the stream's pending work, then wait for the copy itself.
cudaError_t to_dev(kd_batch* b, void* dst, const void* src, size_t bytes) {
  if (!bytes) return cudaSuccess;
  const cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, b->stream);
  return e != cudaSuccess ? e : cudaStreamSynchronize(b->stream);
}
cudaError_t to_host(kd_batch* b, void* dst, const void* src, size_t bytes) {
  if (!bytes) return cudaSuccess;
  const cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, b->stream);
  return e != cudaSuccess ? e : cudaStreamSynchronize(b->stream);
}
}  // namespace

extern "C" {

const char* kd_last_error(void) { return g_err.c_str(); }
const char* kd_version(void) { return "kamino_b200 0.1 (sm_100a)"; }

int kd_abi_sizes(int32_t* out, int32_t cap) {
  const int32_t s[10] = {(int32_t)sizeof(kd_body_desc),   (int32_t)sizeof(kd_joint_desc),
                         (int32_t)sizeof(kd_geom_desc),   (int32_t)sizeof(kd_scene_desc),
                         (int32_t)sizeof(kd_step_config), (int32_t)sizeof(kd_step_diag),
                         (int32_t)sizeof(kd_model_info),  (int32_t)sizeof(kd_row_dump),
                         (int32_t)sizeof(kd_limit_cache_entry), (int32_t)sizeof(kd_contact_cache_entry)};
  const int n = cap < 10 ? cap : 10;
  for (int i = 0; i < n; ++i) out[i] = s[i];
  return n;
}

void kd_step_config_default(kd_step_config* c) {
  c->dt = 1.0 / 240.0;
  c->integrator = KD_INTEGRATOR_SEMI_IMPLICIT_EULER;
  c->backend = KD_BACKEND_AUTO;
  c->eta = 1e-6;
  c->rho = 0.1;
  c->eps = 1e-6;
  c->max_iters = 200;
  c->acceleration = 1;
  c->restart = 1;
  c->fixed_iteration_mode = 0;
  c->cr_iters = 9;
  c->baumgarte_beta = 0.2;
  c->contact_margin = 0.01;
  c->impact_velocity_threshold = 0.1;
  c->bias_clamp = 10.0;
  c->limit_margin_angular = 0.01;
  c->limit_margin_linear = 0.001;
  c->warm_start = 1;
}

int kd_model_build(const kd_scene_desc* scene, kd_model** out) { return kd_model_build_ex(scene, 0, out); }

int kd_model_build_ex(const kd_scene_desc* scene, uint32_t extensions, kd_model** out) {
  if (!scene || !out) return fail(KD_ERR_INVALID_ARGUMENT, "null argument");
  if (extensions & ~KD_EXT_BOX_BOX) return fail(KD_ERR_INVALID_ARGUMENT, "unknown extension bits");
  auto* m = new kd_model;
  std::string err;
  const int code = build_host_model(scene, m->m, err, extensions);
  if (code != KD_OK) {
    delete m;
    return fail(code, err);
  }
  auto plan = std::make_shared<SnPlanHost>();
  if (build_sn_plan(m->m, *plan, m->m.sn_why)) m->m.sn = plan;
  *out = m;
  return KD_OK;
}

int kd_model_sparse_plan_info(const kd_model* mp, int64_t* st) {
  if (!mp || !st) return fail(KD_ERR_INVALID_ARGUMENT, "null argument");
  if (!mp->m.sn) return fail(KD_ERR_INVALID_ARGUMENT, "model has no sparse plan: " + mp->m.sn_why);
  const SnPlanHost& p = *mp->m.sn;
  const int64_t v[14] = {p.S, p.nnzL, p.nLv, (int64_t)p.sup.size(), p.s_levels, (int64_t)p.prog.size(),
                         p.factor_fma, p.solve_terms, p.dense_factor_fma, p.smem_doubles, p.solve_crit, p.n_sph,
                         (int64_t)p.lmask, (int64_t)p.xmask};
  for (int k = 0; k < 14; ++k) st[k] = v[k];
  return KD_OK;
}

int kd_model_sparse_plan_selftest(const kd_model* mp, uint64_t seed, double* max_rel_err) {
  if (!mp || !max_rel_err) return fail(KD_ERR_INVALID_ARGUMENT, "null argument");
  if (!mp->m.sn) return fail(KD_ERR_INVALID_ARGUMENT, "model has no sparse plan: " + mp->m.sn_why);
  const SnPlanHost& p = *mp->m.sn;
  const int S = p.S;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  // rows with random 6-blocks on their slot bodies: D = J J^T + 0.1 I has the plan's pattern
  std::vector<double> J((size_t)S * 12);
  for (double& x : J) x = U(rng);
  std::vector<uint8_t> act(S);
  for (int s = 0; s < S; ++s) act[s] = s < p.n_jd ? 1 : (rng() & 1);
  std::vector<double> D((size_t)S * S, 0.0), b(S), x(S);
  for (int s = 0; s < S; ++s) {
    b[s] = U(rng);
    for (int t = 0; t < S; ++t) {
      double v = s == t ? 0.1 : 0.0;
      for (int u = 0; u < 2; ++u)
        for (int w = 0; w < 2; ++w) {
          const int bs = p.slot_body[2 * s + u];
          if (bs >= 0 && bs == p.slot_body[2 * t + w])
            for (int k = 0; k < 6; ++k) v += J[(size_t)s * 12 + 6 * u + k] * J[(size_t)t * 12 + 6 * w + k];
        }
      D[(size_t)s * S + t] = v;
    }
  }
  if (!sn_plan_cpu_solve(p, D.data(), act.data(), b.data(), x.data()))
    return fail(KD_ERR_SPD_FAILURE, "plan factorization hit a non-positive pivot");
  // dense reference on the active subsystem
  std::vector<int> idx;
  for (int s = 0; s < S; ++s)
    if (act[s]) idx.push_back(s);
  const int n = (int)idx.size();
  std::vector<double> A((size_t)n * n), y(n);
  for (int i = 0; i < n; ++i) {
    y[i] = b[idx[i]];
    for (int j = 0; j < n; ++j) A[(size_t)i * n + j] = D[(size_t)idx[i] * S + idx[j]];
  }
  for (int j = 0; j < n; ++j) {
    double d = A[(size_t)j * n + j];
    for (int k = 0; k < j; ++k) d -= A[(size_t)j * n + k] * A[(size_t)j * n + k];
    d = std::sqrt(d);
    A[(size_t)j * n + j] = d;
    for (int i = j + 1; i < n; ++i) {
      double v = A[(size_t)i * n + j];
      for (int k = 0; k < j; ++k) v -= A[(size_t)i * n + k] * A[(size_t)j * n + k];
      A[(size_t)i * n + j] = v / d;
    }
  }
  for (int i = 0; i < n; ++i) {
    for (int k = 0; k < i; ++k) y[i] -= A[(size_t)i * n + k] * y[k];
    y[i] /= A[(size_t)i * n + i];
  }
  for (int i = n - 1; i >= 0; --i) {
    for (int k = i + 1; k < n; ++k) y[i] -= A[(size_t)k * n + i] * y[k];
    y[i] /= A[(size_t)i * n + i];
  }
  double err = 0.0, scale = 0.0;
  for (int i = 0; i < n; ++i) scale = std::max(scale, std::fabs(y[i]));
  for (int i = 0; i < n; ++i) err = std::max(err, std::fabs(x[idx[i]] - y[i]));
  for (int s = 0; s < S; ++s)
    if (!act[s]) err = std::max(err, std::fabs(x[s]));
  *max_rel_err = err / std::max(scale, 1e-300);
  return KD_OK;
}

void kd_model_destroy(kd_model* m) { delete m; }

int kd_model_set_contact_capacity(kd_model* m, int32_t capacity) {
  if (!m) return fail(KD_ERR_INVALID_ARGUMENT, "null model");
  m->m.contact_cap = capacity > 0 ? std::min(capacity, m->m.info.max_contacts) : 0;
  return KD_OK;
}

int kd_model_get_info(const kd_model* m, kd_model_info* out) {
  if (!m || !out) return fail(KD_ERR_INVALID_ARGUMENT, "null argument");
  *out = m->m.info;
  return KD_OK;
}

int kd_model_joint_layout(const kd_model* mp, int32_t* ro, int32_t* rc, int32_t* dof, int32_t* dc) {
  if (!mp) return fail(KD_ERR_INVALID_ARGUMENT, "null model");
  const HostModel& m = mp->m;
  for (size_t j = 0; j < m.joints.size(); ++j) {
    const DevJoint& J = m.joints[j];
    ro[j] = J.row_offset;
    rc[j] = J.row_count;
    dof[j] = J.dyn_offset;
    dc[j] = ((J.flags & JF_PD) ? 1 : 0) + ((J.flags & JF_ARMATURE) ? 1 : 0) + ((J.flags & JF_DAMPING) ? 1 : 0);
  }
  return KD_OK;
}

int kd_model_joint_targets(const kd_model* mp, double* t) {
  if (!mp) return fail(KD_ERR_INVALID_ARGUMENT, "null model");
  for (size_t j = 0; j < mp->m.joints.size(); ++j) t[j] = mp->m.joints[j].target;
  return KD_OK;
}

int kd_joint_coordinate(const kd_model* mp, int32_t joint, const double* poses7, double* out) {
  if (!mp || !poses7 || !out) return fail(KD_ERR_INVALID_ARGUMENT, "null argument");
  const HostModel& m = mp->m;
  if (joint < 0 || joint >= (int)m.joints.size()) return fail(KD_ERR_INVALID_ARGUMENT, "joint index out of range");
  const int t = m.joints[joint].type;
  if (t != J_REVOLUTE && t != J_PRISMATIC)
    return fail(KD_ERR_MODEL_WRONG_JOINT_TYPE, "joint '" + m.joint_names[joint] + "' has no scalar coordinate");
  *out = host_joint_coordinate(m, joint, poses7);
  return KD_OK;
}

// --------------------------------------------------------------------- batch
int kd_batch_create(int32_t device, const kd_model* const* models, int32_t n_models, const int32_t* world_model,
                    int32_t n_worlds, kd_batch** out) {
  // an empty batch (no models, no worlds) is valid, as WorldBatch() is (batch.hpp:14-54)
  if (!out || n_models < 0 || (n_models > 0 && !models) || n_worlds < 0 || (n_worlds > 0 && (!world_model || n_models == 0)))
    return fail(KD_ERR_INVALID_ARGUMENT, "invalid arguments");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(KD_ERR_NO_DEVICE, "no CUDA device visible: the B200 solver has no CPU fallback");
  if (device < 0 || device >= ndev) return fail(KD_ERR_INVALID_ARGUMENT, "device index out of range");
  KD_CK(cudaSetDevice(device));
  auto* b = new kd_batch;
  std::unique_ptr<kd_batch> guard(b);
  b->device = device;
  KD_CK(cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking));
  for (int i = 0; i < n_models; ++i) {
    if (!models[i]) return fail(KD_ERR_INVALID_ARGUMENT, "null model");
    b->models.push_back(models[i]->m);
  }
  {  // supernodal path: KD_SPARSE=0 off, 1 (default) for small planned models, 2 for every planned model
    const char* e = getenv("KD_SPARSE");
    b->sparse_mode = e ? (e[0] == '0' ? 0 : (e[0] == '2' ? 2 : 1)) : 1;
    b->sparse = b->sparse_mode != 0;
    const char* h = getenv("KD_SN_HANDOFF");
    b->sn_handoff = !(h && h[0] == '0');
    const char* g = getenv("KD_GRAPHS");  // KD_GRAPHS=0: launch every kernel directly
    b->graphs = !(g && g[0] == '0');
    const char* df = getenv("KD_DENSE_DF");  // KD_DENSE_DF=0: barrier between the dense solve passes
    b->no_df = df && df[0] == '0';
    const char* tme = getenv("KD_TMEM");  // KD_TMEM=0: the dense solve reads X's tiles from shared memory only
    b->no_tmem = tme && tme[0] == '0';
    const char* cle = getenv("KD_CLUSTER");  // KD_CLUSTER=1: the opt-in K2c path (kd_dense_cl.cu)
    b->cluster = cle && cle[0] == '1';
  }
  b->n_worlds = n_worlds;
  // model tables
  std::vector<DevModel> dm(n_models);
  std::vector<DevBody> bodies;
  std::vector<DevJoint> joints;
  std::vector<DevGeom> geoms;
  std::vector<DevPair> pairs;
  std::vector<int> contact_cap(n_models), row_cap(n_models);
  for (int i = 0; i < n_models; ++i) {
    const HostModel& m = b->models[i];
    DevModel& d = dm[i];
    d.nb = (int)m.bodies.size();
    d.nj = (int)m.joints.size();
    d.ng = (int)m.geoms.size();
    d.npairs = (int)m.pairs.size();
    d.n_bil = m.n_bil;
    d.n_dyn = m.n_dyn;
    d.n_limited = m.info.n_limited_joints;
    // contact capacity: every supported pair can produce 1 (4 for box-plane and
    // box-box) contact, capped for large piles at 6 per geom (8 with box-box
    // pairs: face contacts carry 4 points) + 16; overflow is an error.
    bool box_box = false;
    for (const DevPair& pr : m.pairs) box_box = box_box || pr.kind == P_BOX_BOX;
    contact_cap[i] = m.contact_cap > 0 ? std::min(m.info.max_contacts, m.contact_cap)
                                       : std::min(m.info.max_contacts, (box_box ? 8 : 6) * d.ng + 16);
    d.max_contacts = contact_cap[i];
    row_cap[i] = d.n_bil + d.n_dyn + 2 * d.n_limited + 3 * contact_cap[i];
    d.row_cap = row_cap[i];
    d.body_off = (int)bodies.size();
    d.joint_off = (int)joints.size();
    d.geom_off = (int)geoms.size();
    d.pair_off = (int)pairs.size();
    // Auto: the supernodal kernel (a warp per world, several worlds per CTA)
    // wins on small systems (measured 2.1x on fourbar, 1.9x on double_fourbar);
    // on larger ones (serial_chain_10, DR-Legs) the fused dense kernel's
    // parallel explicit-inverse solves win (tests/kernel_ab.py).
    // Larger planned models (S <= the dense kernel's shared-memory rows) use
    // the hand-off: the supernodal kernel factors D in the plan's order (38k
    // FMA instead of 1.8M for DR-Legs, several worlds per SM) and the dense
    // kernel forms L^-1 and runs the PADMM solves (KD_SN_HANDOFF=0 disables).
    const bool sn_fits =
        m.sn && (size_t)m.sn->smem_doubles * 8 + (((size_t)m.sn->prog.size() * 4 + 15) & ~(size_t)15) <= kSnMaxSmem;
    d.sn = 0;
    if (b->sparse && sn_fits) {
      if (b->sparse_mode == 2 || m.sn->S <= kSnAutoMaxSlots) d.sn = 1;
      else if (b->sn_handoff && m.sn->S <= kSmemMaxRows && !m.sn->scat.empty()) d.sn = 2;
    }
    for (int k = 0; k < 3; ++k) d.gravity[k] = m.gravity[k];
    if (i == 0) {
      b->cl_split.assign(n_models, 0);
      b->cl_xlen.assign(n_models, 0);
    }
    if (d.sn == 2 && b->cluster && m.sn->S <= 256 && m.sn->xmask != ~0ull && row_cap[i] > kClasses[2][0]) {
      // tile rows [0, k) to CTA 0, [k, T) to CTA 1: the split with the
      // smaller larger half whose CTAs both fit twice per SM
      const int T = (m.sn->S + 31) / 32;
      std::vector<int> rlen(T, 0), ritems(T, 0);
      for (int ti = 0; ti < T; ++ti)
        for (int tj = 0; tj <= ti; ++tj)
          if ((m.sn->xmask >> (ti * (ti + 1) / 2 + tj)) & 1ull) {
            rlen[ti] += ti == tj ? 528 : 32 * 33;
            ++ritems[ti];
          }
      int items = 0, xlen = 0;
      for (int ti = 0; ti < T; ++ti) {
        items += ritems[ti];
        xlen += rlen[ti];
      }
      int best = 0;
      size_t best_bytes = 0;
      int l0 = 0;
      for (int k = 1; k < T; ++k) {
        l0 += rlen[k - 1];
        const int own = std::max(l0, xlen - l0);
        const size_t bytes = dense_cl_smem_bytes(own, items, T);
        if (bytes + dense_cl_static_bytes() + 1024 <= kClPerCta && (!best || bytes < best_bytes)) {
          best = k;
          best_bytes = bytes;
        }
      }
      if (best) {
        b->cl_split[i] = best;
        b->cl_xlen[i] = xlen;
        b->cl_smem = std::max(b->cl_smem, best_bytes);
      }
    }
    bodies.insert(bodies.end(), m.bodies.begin(), m.bodies.end());
    joints.insert(joints.end(), m.joints.begin(), m.joints.end());
    geoms.insert(geoms.end(), m.geoms.begin(), m.geoms.end());
    pairs.insert(pairs.end(), m.pairs.begin(), m.pairs.end());
  }
  // world layout
  b->world_model.assign(world_model, world_model + n_worlds);
  b->worlds.resize(n_worlds);
  b->pose_off.resize(n_worlds);
  b->twist_off.resize(n_worlds);
  b->row_off.resize(n_worlds);
  std::vector<double> h_pose, h_twist;
  std::vector<std::vector<int32_t>> class_worlds(4);
  for (int w = 0; w < n_worlds; ++w) {
    const int mi = world_model[w];
    if (mi < 0 || mi >= n_models) return fail(KD_ERR_INVALID_ARGUMENT, "world_model index out of range");
    const HostModel& m = b->models[mi];
    DevWorld& W = b->worlds[w];
    W.model = mi;
    W.nb = (int)m.bodies.size();
    W.pose_off = (int)b->pose_len;
    W.twist_off = (int)b->twist_len;
    W.row_off = b->total_rows;
    W.body_off = b->total_bodies;
    W.contact_off = b->total_contacts;
    W.jcache_off = b->total_jcache;
    W.lslot_off = b->total_lslots;
    W.contact_cap = contact_cap[mi];
    const int rc = row_cap[mi];
    int cls = 3;
    for (int c = 0; c < 4; ++c)
      if (std::min(rc, kSmemMaxRows) <= kClasses[c][0]) {
        cls = c;
        break;
      }
    W.bin = cls;
    W.smem_cap = kClasses[cls][0];
    class_worlds[cls].push_back(w);
    W.slab_cap = 0;
    W.lslab_off = -1;
    W.snlv_off = -1;
    W.snr2p_off = -1;
    W.xslab_off = -1;
    if (b->cl_split[mi]) {
      W.xslab_off = b->total_xslab;
      b->total_xslab += b->cl_xlen[mi];
    }
    if (dm[mi].sn == 2) {
      W.snlv_off = b->total_snlv;
      b->total_snlv += (m.sn->nLv + 1) & ~1;
      W.snr2p_off = b->total_snr2p;
      b->total_snr2p += m.sn->S;
    }
    if (rc > kSmemMaxRows) {
      W.slab_cap = std::min(rc, kDenseGlobalMaxRows);
      W.lslab_off = b->total_lslab;
      b->total_lslab += slab_doubles(W.slab_cap);
      b->global_bin.worlds.push_back(w);
      b->global_bin.cap = std::max(b->global_bin.cap, W.slab_cap);
      b->has_big = b->has_big || rc > kDenseGlobalMaxRows;
    }
    if (rc > kDenseGlobalMaxRows) {
      b->cr_auto_bin.worlds.push_back(w);
      b->cr_auto_bin.cap = std::max(b->cr_auto_bin.cap, rc);
      b->cr_auto_bin.nbcap = std::max(b->cr_auto_bin.nbcap, W.nb);
    }
    b->cr_all_bin.worlds.push_back(w);
    b->cr_all_bin.cap = std::max(b->cr_all_bin.cap, rc);
    b->cr_all_bin.nbcap = std::max(b->cr_all_bin.nbcap, W.nb);
    b->pose_off[w] = W.pose_off;
    b->twist_off[w] = W.twist_off;
    b->row_off[w] = W.row_off;
    b->pose_len += 7 * W.nb;
    b->twist_len += 6 * W.nb;
    b->total_rows += rc;
    b->total_bodies += W.nb;
    b->total_contacts += contact_cap[mi];
    b->total_jcache += m.n_bil + m.n_dyn;
    b->total_lslots += 2 * m.info.n_limited_joints;
    h_pose.insert(h_pose.end(), m.init_pose.begin(), m.init_pose.end());
    h_twist.insert(h_twist.end(), m.init_twist.begin(), m.init_twist.end());
  }
  // models whose worlds always take their plan's kernel under a dense choice:
  // K2s end to end (sn == 1) never reaches the dense bins, the hand-off
  // (sn == 2) runs in them but never in the HBM-slab bin
  std::vector<int> always_planned(n_models, 0);
  for (int i = 0; i < n_models; ++i) {
    const auto* pl = b->models[i].sn.get();
    bool all = dm[i].sn != 0 && pl;
    if (all)
      for (int32_t ps : pl->pair_slot) all = all && ps >= 0;
    always_planned[i] = all ? dm[i].sn : 0;
  }
  for (int c = 0; c < 4; ++c) {
    if (class_worlds[c].empty()) continue;
    Bin bin;
    bin.cap = kClasses[c][0];
    bin.nt = kClasses[c][1];
    bin.worlds = class_worlds[c];
    bin.never = true;
    for (int32_t w : bin.worlds) bin.never = bin.never && always_planned[world_model[w]] == 1;
    b->dense_bins.push_back(bin);
  }
  b->global_bin.never = true;
  {
    const char* sw = getenv("KD_SLAB_SWEEP");  // KD_SLAB_SWEEP=1: every slab bin through the sweep kernel (tests)
    b->global_bin.rare = true;
    b->slab_sweep_forced = sw && sw[0] == '1';
  }
  for (int32_t w : b->global_bin.worlds) {
    b->global_bin.never = b->global_bin.never && always_planned[world_model[w]] != 0;
    b->global_bin.rare = b->global_bin.rare && dm[world_model[w]].sn != 0;
  }
  for (int i = 0; i < n_models; ++i) {
    if (!dm[i].sn) continue;
    kd_batch::SnBin sbn;
    sbn.model = i;
    sbn.hand = dm[i].sn == 2;  // hand-off: the factor kernel K2f, then the dense kernel
    sbn.hand_smem = snfactor_smem_bytes(b->models[i].sn->nLv, b->models[i].sn->S);
    sbn.per_warp = b->models[i].sn->smem_doubles;
    sbn.prog_words = (int)b->models[i].sn->prog.size();
    const size_t prog_bytes = ((size_t)sbn.prog_words * 4 + 15) & ~(size_t)15;
    sbn.wpc = (int)std::max<size_t>(1, std::min<size_t>(8, (kSnMaxSmem - prog_bytes) / (8 * (size_t)sbn.per_warp)));
    for (int w = 0; w < n_worlds; ++w)
      if (world_model[w] == i) sbn.bin.worlds.push_back(w);
    if (!sbn.bin.worlds.empty()) b->sn_bins.push_back(sbn);
  }
  b->global_bin.nt = 256;
  for (Bin* bin : {&b->cr_auto_bin, &b->cr_all_bin}) bin->nt = bin->cap > 256 ? 512 : (bin->cap > 128 ? 256 : 128);

  // device allocations
  BatchView& v = b->view;
  DevMem& mem = b->mem;
  const int64_t R = std::max<int64_t>(1, b->total_rows);
  DevModel* d_models;
  DevBody* d_bodies;
  DevJoint* d_joints;
  DevGeom* d_geoms;
  DevPair* d_pairs;
  DevWorld* d_worlds;
  uint8_t* d_active;
  KD_CK(mem.alloc(d_models, n_models));
  KD_CK(mem.alloc(d_bodies, bodies.size()));
  KD_CK(mem.alloc(d_joints, joints.size()));
  KD_CK(mem.alloc(d_geoms, geoms.size()));
  KD_CK(mem.alloc(d_pairs, pairs.size()));
  KD_CK(mem.alloc(d_worlds, n_worlds));
  KD_CK(mem.alloc(d_active, n_worlds));
  KD_CK(cudaMemcpy(d_models, dm.data(), sizeof(DevModel) * dm.size(), cudaMemcpyHostToDevice));
  if (!bodies.empty()) KD_CK(cudaMemcpy(d_bodies, bodies.data(), sizeof(DevBody) * bodies.size(), cudaMemcpyHostToDevice));
  if (!joints.empty()) KD_CK(cudaMemcpy(d_joints, joints.data(), sizeof(DevJoint) * joints.size(), cudaMemcpyHostToDevice));
  if (!geoms.empty()) KD_CK(cudaMemcpy(d_geoms, geoms.data(), sizeof(DevGeom) * geoms.size(), cudaMemcpyHostToDevice));
  if (!pairs.empty()) KD_CK(cudaMemcpy(d_pairs, pairs.data(), sizeof(DevPair) * pairs.size(), cudaMemcpyHostToDevice));
  if (n_worlds) KD_CK(cudaMemcpy(d_worlds, b->worlds.data(), sizeof(DevWorld) * n_worlds, cudaMemcpyHostToDevice));
  {
    std::vector<uint8_t> ones(std::max(1, n_worlds), 1);
    KD_CK(cudaMemcpy(d_active, ones.data(), std::max(1, n_worlds), cudaMemcpyHostToDevice));
  }
  v.n_worlds = n_worlds;
  v.models = d_models;
  v.bodies = d_bodies;
  v.joints = d_joints;
  v.geoms = d_geoms;
  v.pairs = d_pairs;
  v.worlds = d_worlds;
  v.active = d_active;
  KD_CK(mem.alloc(v.poses, b->pose_len));
  KD_CK(mem.alloc(v.twists, b->twist_len));
  KD_CK(mem.alloc(v.time, n_worlds));
  KD_CK(mem.alloc(v.wstep, n_worlds));
  KD_CK(mem.alloc(v.rowj, R));
  KD_CK(mem.alloc(v.rbody, 2 * R));
  KD_CK(mem.alloc(v.rkind, R));
  KD_CK(mem.alloc(v.lkey, 2 * R));
  KD_CK(mem.alloc(v.rmu, R));
  KD_CK(mem.alloc(v.bias, R));
  KD_CK(mem.alloc(v.reg, R));
  KD_CK(mem.alloc(v.scale, R));
  KD_CK(mem.alloc(v.vf, R));
  KD_CK(mem.alloc(v.x0, R));
  KD_CK(mem.alloc(v.z0, R));
  KD_CK(mem.alloc(v.lam, R));
  KD_CK(mem.alloc(v.zo, R));
  KD_CK(mem.alloc(v.imp, R));
  KD_CK(mem.alloc(v.csr_ptr, b->total_bodies + n_worlds));
  KD_CK(mem.alloc(v.csr, 2 * R));
  KD_CK(mem.alloc(v.bs, b->total_bodies));
  KD_CK(mem.alloc(v.contacts, b->total_contacts));
  KD_CK(mem.alloc(v.ccache, b->total_contacts));
  KD_CK(mem.alloc(v.jc_lam, b->total_jcache));
  KD_CK(mem.alloc(v.jc_z, b->total_jcache));
  KD_CK(mem.alloc(v.ls_lam, b->total_lslots));
  KD_CK(mem.alloc(v.ls_z, b->total_lslots));
  KD_CK(mem.alloc(v.ls_valid, b->total_lslots));
  KD_CK(mem.alloc(v.lslab, b->total_lslab));
  KD_CK(mem.alloc(v.sn_lv, b->total_snlv));
  if (b->total_xslab && mem.alloc(v.xslab, b->total_xslab) != cudaSuccess) {
    cudaGetLastError();  // no room for the K2c slab: K2 keeps the PADMM of every world
    b->total_xslab = 0;
    b->cl_smem = 0;
    for (DevWorld& W : b->worlds) W.xslab_off = -1;
    KD_CK(cudaMemcpy(d_worlds, b->worlds.data(), sizeof(DevWorld) * n_worlds, cudaMemcpyHostToDevice));
  }
  KD_CK(mem.alloc(v.sn_r2p, b->total_snr2p));
  if (cr_smem_bytes(b->cr_all_bin.cap, b->cr_all_bin.nbcap, 512) > 232448) {
    // worlds too large for one CTA's shared memory: the shared CR kernel keeps
    // its vectors (and the staged P J) in a per-world HBM slab instead
    const int64_t stride = (int64_t)((cr_staged_bytes(b->cr_all_bin.cap, b->cr_all_bin.nbcap, 512) + 15) / 16 * 2);
    if (mem.alloc(v.cr_scratch, (size_t)stride * std::max(1, n_worlds)) != cudaSuccess) {
      cudaGetLastError();
      return fail(KD_ERR_CAPACITY, "matrix-free path: the per-world scratch of worlds beyond one CTA's shared memory "
                                   "does not fit device memory");
    }
    v.cr_scratch_stride = stride;
  }
  KD_CK(mem.alloc(b->d_hist, 1));
  KD_CK(mem.alloc(b->d_err, 4));
  v.hist = b->d_hist;
  v.hist_cap = 0;
  v.error_count = b->d_err;
  if (b->pose_len) KD_CK(cudaMemcpy(v.poses, h_pose.data(), 8 * b->pose_len, cudaMemcpyHostToDevice));
  if (b->twist_len) KD_CK(cudaMemcpy(v.twists, h_twist.data(), 8 * b->twist_len, cudaMemcpyHostToDevice));
  {
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    const char* e = getenv("KD_SPLIT");
    int np = e ? std::max(1, std::min(4, atoi(e))) : 2;
    const char* em = getenv("KD_SPLIT_MIN");  // worlds per part at least (default 8 per SM)
    const int per = em ? std::max(1, atoi(em)) : 8 * nsm;
    while (np > 1 && n_worlds < per * np) --np;  // every part still fills the GPU
    b->n_halves = np;
    for (int p = 0; p <= np; ++p) b->cut[p] = (int)((int64_t)n_worlds * p / np);
    b->pstream[0] = b->stream;
    if (np > 1) KD_CK(cudaEventCreateWithFlags(&b->ev_fork, cudaEventDisableTiming));
    for (int p = 1; p < np; ++p) {
      KD_CK(cudaStreamCreateWithFlags(&b->pstream[p], cudaStreamNonBlocking));
      KD_CK(cudaEventCreateWithFlags(&b->ev_join[p], cudaEventDisableTiming));
    }
  }
  for (Bin* bin : {&b->global_bin, &b->cr_auto_bin, &b->cr_all_bin}) bin->set_parts(b->cut, b->n_halves);
  for (Bin& bin : b->dense_bins) bin.set_parts(b->cut, b->n_halves);
  for (auto& sbn : b->sn_bins) sbn.bin.set_parts(b->cut, b->n_halves);
  for (Bin* bin : {&b->global_bin, &b->cr_auto_bin, &b->cr_all_bin}) {
    bin->count = (int)bin->worlds.size();
    if (bin->count) {
      KD_CK(mem.alloc(bin->d_worlds, bin->count));
      KD_CK(cudaMemcpy(bin->d_worlds, bin->worlds.data(), 4 * bin->count, cudaMemcpyHostToDevice));
    }
  }
  for (Bin& bin : b->dense_bins) {
    bin.count = (int)bin.worlds.size();
    KD_CK(mem.alloc(bin.d_worlds, bin.count));
    KD_CK(cudaMemcpy(bin.d_worlds, bin.worlds.data(), 4 * bin.count, cudaMemcpyHostToDevice));
  }
  for (auto& sbn : b->sn_bins) {
    sbn.bin.count = (int)sbn.bin.worlds.size();
    KD_CK(mem.alloc(sbn.bin.d_worlds, sbn.bin.count));
    KD_CK(cudaMemcpy(sbn.bin.d_worlds, sbn.bin.worlds.data(), 4 * sbn.bin.count, cudaMemcpyHostToDevice));
  }
  {  // supernodal plans, concatenated over models with relocated offsets
    std::vector<DevSnPlan> dp(n_models);
    std::vector<SnGram> gram;
    std::vector<SnSuper> sups;
    std::vector<int32_t> prow;
    std::vector<uint32_t> scat;
    std::vector<SnGBody> gbody;
    std::vector<uint32_t> tmap, prog, gslot, gpair;
    std::vector<int32_t> pslot;
    std::vector<uint16_t> spos;
    std::vector<uint8_t> kmask;
    for (int i = 0; i < n_models; ++i) {
      DevSnPlan& d = dp[i];
      d = DevSnPlan{};
      if (!dm[i].sn) continue;
      const SnPlanHost& p = *b->models[i].sn;
      d.S = p.S;
      d.nLv = p.nLv;
      d.n_jd = p.n_jd;
      d.lim_base = p.lim_base;
      d.smem_doubles = p.smem_doubles;
      d.max_slots = p.max_slots;
      d.lmask_lo = (int32_t)(uint32_t)(p.lmask & 0xffffffffull);
      d.lmask_hi = (int32_t)(uint32_t)(p.lmask >> 32);
      d.xmask_lo = (int32_t)(uint32_t)(p.xmask & 0xffffffffull);
      d.xmask_hi = (int32_t)(uint32_t)(p.xmask >> 32);
      d.cl_split = b->cl_split[i];
      d.cl_xlen = b->cl_xlen[i];
      d.kmask_off = (int)kmask.size();
      kmask.insert(kmask.end(), p.kmask.begin(), p.kmask.end());
      d.n_sph = p.n_sph;
      d.gram_off = (int)gram.size();
      d.n_gram = (int)p.gram.size();
      gram.insert(gram.end(), p.gram.begin(), p.gram.end());
      d.pair_off = (int)pslot.size();
      pslot.insert(pslot.end(), p.pair_slot.begin(), p.pair_slot.end());
      d.slotpos_off = (int)spos.size();
      spos.insert(spos.end(), p.slot_pos.begin(), p.slot_pos.end());
      d.kmax = p.kmax;
      d.vreg = p.vreg;
      d.gbody_off = (int)gbody.size();
      d.n_gbody = (int)p.gbody.size();
      {
        const int so = (int)gslot.size(), po = (int)gpair.size();
        for (SnGBody g : p.gbody) {
          g.slot_off += so;
          g.pair_off += po;
          gbody.push_back(g);
        }
        gslot.insert(gslot.end(), p.gslot.begin(), p.gslot.end());
        gpair.insert(gpair.end(), p.gpair.begin(), p.gpair.end());
      }
      d.sup_off = (int)sups.size();
      d.n_sup = (int)p.sup.size();
      const int to = (int)tmap.size(), po = (int)prow.size();
      for (SnSuper u : p.sup) {
        u.tmap_off += to;
        u.prow_off += po;
        sups.push_back(u);
      }
      prow.insert(prow.end(), p.prow.begin(), p.prow.end());
      d.scat_off = (int)scat.size();
      d.n_scat = (int)p.scat.size();
      scat.insert(scat.end(), p.scat.begin(), p.scat.end());
      tmap.insert(tmap.end(), p.tmap.begin(), p.tmap.end());
      while (prog.size() & 3) prog.push_back(0);  // 16-byte aligned blobs
      d.prog_off = (int)prog.size();
      d.prog_words = (int)p.prog.size();
      prog.insert(prog.end(), p.prog.begin(), p.prog.end());
    }
    auto up = [&](auto*& dst, const auto& vec) -> cudaError_t {
      using T = typename std::remove_reference<decltype(vec)>::type::value_type;
      T* ptr = nullptr;
      cudaError_t e = mem.alloc(ptr, vec.size());
      if (e == cudaSuccess && !vec.empty()) e = cudaMemcpy(ptr, vec.data(), sizeof(T) * vec.size(), cudaMemcpyHostToDevice);
      dst = ptr;
      return e;
    };
    KD_CK(up(v.snplan, dp));
    KD_CK(up(v.sn_gram, gram));
    KD_CK(up(v.sn_gbody, gbody));
    KD_CK(up(v.sn_gslot, gslot));
    KD_CK(up(v.sn_gpair, gpair));
    KD_CK(up(v.sn_sup, sups));
    KD_CK(up(v.sn_tmap, tmap));
    KD_CK(up(v.sn_prog, prog));
    KD_CK(up(v.sn_pair_slot, pslot));
    KD_CK(up(v.sn_slot_pos, spos));
    KD_CK(up(v.sn_prow, prow));
    KD_CK(up(v.sn_scat, scat));
    KD_CK(up(v.sn_kmask, kmask));
  }
  for (cudaEvent_t& e : b->ev) KD_CK(cudaEventCreate(&e));
  // the uploads above ran on the legacy stream: wait for it alone (a device-wide
  // synchronize would fail while another host thread captures a step graph)
  KD_CK(cudaStreamSynchronize(0));
  *out = guard.release();
  return KD_OK;
}

void kd_batch_destroy(kd_batch* b) {
  if (!b) return;
  cudaSetDevice(b->device);
  delete b;
}

int kd_batch_size(const kd_batch* b, int32_t* nw, int64_t* pl, int64_t* tl) {
  if (!b) return fail(KD_ERR_INVALID_ARGUMENT, "null batch");
  if (nw) *nw = b->n_worlds;
  if (pl) *pl = b->pose_len;
  if (tl) *tl = b->twist_len;
  return KD_OK;
}

int kd_batch_offsets(const kd_batch* b, int32_t* po, int32_t* to) {
  if (!b) return fail(KD_ERR_INVALID_ARGUMENT, "null batch");
  for (int w = 0; w < b->n_worlds; ++w) {
    if (po) po[w] = b->pose_off[w];
    if (to) to[w] = b->twist_off[w];
  }
  return KD_OK;
}

int kd_batch_set_state(kd_batch* b, const double* poses, const double* twists, const double* time) {
  if (!b) return fail(KD_ERR_INVALID_ARGUMENT, "null batch");
  KD_CK(cudaSetDevice(b->device));
  if (poses && b->pose_len) KD_CK(to_dev(b, b->view.poses, poses, 8 * b->pose_len));
  if (twists && b->twist_len) KD_CK(to_dev(b, b->view.twists, twists, 8 * b->twist_len));
  if (time && b->n_worlds) KD_CK(to_dev(b, b->view.time, time, 8 * b->n_worlds));
  return KD_OK;
}

int kd_batch_get_state(kd_batch* b, double* poses, double* twists, double* time) {
  if (!b) return fail(KD_ERR_INVALID_ARGUMENT, "null batch");
  KD_CK(cudaSetDevice(b->device));
  KD_CK(cudaStreamSynchronize(b->stream));
  if (poses && b->pose_len) KD_CK(to_host(b, poses, b->view.poses, 8 * b->pose_len));
  if (twists && b->twist_len) KD_CK(to_host(b, twists, b->view.twists, 8 * b->twist_len));
  if (time && b->n_worlds) KD_CK(to_host(b, time, b->view.time, 8 * b->n_worlds));
  return KD_OK;
}

int kd_batch_reset_caches(kd_batch* b) {
  if (!b) return fail(KD_ERR_INVALID_ARGUMENT, "null batch");
  KD_CK(cudaSetDevice(b->device));
  std::vector<WorldStep> ws(b->n_worlds);
  if (b->n_worlds) {
    KD_CK(to_host(b, ws.data(), b->view.wstep, sizeof(WorldStep) * b->n_worlds));
    for (WorldStep& s : ws) {
      s.jcache_valid = 0;
      s.ccache_count = 0;
    }
    KD_CK(to_dev(b, b->view.wstep, ws.data(), sizeof(WorldStep) * b->n_worlds));
  }
  if (b->total_lslots) {
    KD_CK(cudaMemsetAsync(b->view.ls_valid, 0, 4 * b->total_lslots, b->stream));
    KD_CK(cudaStreamSynchronize(b->stream));
  }
  return KD_OK;
}

int kd_batch_set_active(kd_batch* b, const uint8_t* active) {
  if (!b || !active) return fail(KD_ERR_INVALID_ARGUMENT, "null argument");
  KD_CK(cudaSetDevice(b->device));
  if (b->n_worlds)
    KD_CK(to_dev(b, const_cast<uint8_t*>(b->view.active), active, b->n_worlds));
  return KD_OK;
}

int kd_batch_set_history_capacity(kd_batch* b, int32_t cap) {
  if (b) b->drop_graph();  // the captured kernels hold the old history pointer
  if (!b || cap < 0) return fail(KD_ERR_INVALID_ARGUMENT, "invalid argument");
  KD_CK(cudaSetDevice(b->device));
  double* h = nullptr;
  KD_CK(b->mem.alloc(h, (size_t)std::max(1, cap) * std::max(1, b->n_worlds)));
  b->d_hist = h;
  b->hist_cap = cap;
  b->view.hist = h;
  b->view.hist_cap = cap;
  return KD_OK;
}

int kd_batch_get_history(kd_batch* b, double* out) {
  if (!b || !out) return fail(KD_ERR_INVALID_ARGUMENT, "null argument");
  KD_CK(cudaSetDevice(b->device));
  if (b->hist_cap && b->n_worlds)
    KD_CK(to_host(b, out, b->d_hist, 8 * (size_t)b->hist_cap * b->n_worlds));
  return KD_OK;
}

// Per step and kernel family: the span from the family's first start to its
// last end over the batch's parts (parts overlap in time, so a family's span is
// its active wall time; with one part it is the family's own duration).  Part
// 0's first mark precedes the fork, so every other event follows it.
static int resolve_timing(kd_batch* b) {
  if (b->ev_done == b->ev_used) return KD_OK;
  for (int p = 0; p < b->n_halves; ++p) KD_CK(cudaStreamSynchronize(b->pstream[p]));
  const size_t per = 5 * (size_t)b->n_halves;
  for (size_t k = b->ev_done; k < b->ev_used; k += per) {
    float t[4][5];
    for (int p = 0; p < b->n_halves; ++p)
      for (int i = 0; i < 5; ++i) {
        t[p][i] = 0.f;
        if (p || i) KD_CK(cudaEventElapsedTime(&t[p][i], b->evpool[k], b->evpool[k + 5 * p + i]));
      }
    for (int i = 0; i < 4; ++i) {
      float lo = t[0][i], hi = t[0][i + 1];
      for (int p = 1; p < b->n_halves; ++p) {
        lo = std::min(lo, t[p][i]);
        hi = std::max(hi, t[p][i + 1]);
      }
      b->ms[i] += hi - lo;
    }
  }
  b->ev_done = b->ev_used = 0;
  return KD_OK;
}

int kd_batch_enable_timing(kd_batch* b, int32_t on) {
  if (!b) return fail(KD_ERR_INVALID_ARGUMENT, "null batch");
  KD_CK(cudaSetDevice(b->device));
  const int rc = resolve_timing(b);
  if (rc != KD_OK) return rc;
  b->timing = on != 0;
  for (double& m : b->ms) m = 0.0;
  b->launches = 0;
  return KD_OK;
}

int kd_batch_get_timing(kd_batch* b, double* ms4, int64_t* launches) {
  if (!b) return fail(KD_ERR_INVALID_ARGUMENT, "null batch");
  KD_CK(cudaSetDevice(b->device));
  const int rc = resolve_timing(b);
  if (rc != KD_OK) return rc;
  if (ms4)
    for (int i = 0; i < 4; ++i) ms4[i] = b->ms[i];
  if (launches) *launches = b->launches;
  return KD_OK;
}

static StepParams step_params(const kd_batch* b, const kd_step_config* c) {
  StepParams sp{};
  sp.dt = c->dt;
  sp.eta = c->eta;
  sp.rho = c->rho;
  sp.eps = c->eps;
  sp.beta = c->baumgarte_beta;
  sp.contact_margin = c->contact_margin;
  sp.impact_thr = c->impact_velocity_threshold;
  sp.bias_clamp = c->bias_clamp;
  sp.lim_margin_ang = c->limit_margin_angular;
  sp.lim_margin_lin = c->limit_margin_linear;
  sp.max_iters = c->max_iters;
  sp.acceleration = c->acceleration;
  sp.restart = c->restart;
  sp.fixed_mode = c->fixed_iteration_mode;
  sp.cr_iters = c->cr_iters;
  sp.warm_start = c->warm_start;
  sp.moreau = c->integrator == KD_INTEGRATOR_MOREAU_JEAN;
  sp.backend = c->backend;
  sp.sparse = b->sparse ? 1 : 0;
  sp.sn_handoff = b->sn_handoff ? 1 : 0;
  sp.eta_rho = c->eta + c->rho;
  sp.no_df = b->no_df ? 1 : 0;
  sp.no_tmem = b->no_tmem ? 1 : 0;
  sp.nest_beta = b->d_nest;
  return sp;
}

// One step's launches: K1 -> K2s bins -> K2 bins -> K2g -> K2b -> K3.
static int enqueue_one(kd_batch* b, const kd_step_config* c, const StepParams& sp) {
  const BatchView& v = b->view;
  if (b->timing) {
    while (b->evpool.size() < b->ev_used + 5 * (size_t)b->n_halves) {
      cudaEvent_t e;
      KD_CK(cudaEventCreate(&e));
      b->evpool.push_back(e);
    }
  }
  if (b->timing) KD_CK(cudaEventRecord(b->evpool[b->ev_used], b->stream));  // part 0's mark 0, before the fork
  if (b->n_halves > 1) {  // fork: the parts' streams wait for everything before this step
    KD_CK(cudaEventRecord(b->ev_fork, b->stream));
    for (int p = 1; p < b->n_halves; ++p) KD_CK(cudaStreamWaitEvent(b->pstream[p], b->ev_fork, 0));
  }
  for (int h = 0; h < b->n_halves; ++h) {
    cudaStream_t s = b->pstream[h];
    const int w0 = b->cut[h], w1 = b->cut[h + 1];
    const size_t eb = b->ev_used + 5 * (size_t)h;
    auto mark = [&](int i) {
      if (b->timing) cudaEventRecord(b->evpool[eb + i], s);
    };
    auto part = [&](const Bin& bin, int& cnt) -> const int32_t* {
      cnt = bin.hcount[h];
      return bin.d_worlds + bin.hoff[h];
    };
    int cnt = 0;
    if (h) mark(0);
    launch_assemble(v, sp, s, w0, w1);
    KD_CK(cudaGetLastError());
    ++b->launches;
    mark(1);
    if (c->backend != KD_BACKEND_MATRIX_FREE) {
      for (const auto& sbn : b->sn_bins) {
        const int32_t* wl = part(sbn.bin, cnt);
        if (!cnt) continue;
        if (sbn.hand) KD_CK(launch_snfactor(v, sp, wl, cnt, sbn.hand_smem, s));
        else KD_CK(launch_sparse(v, sp, wl, cnt, sbn.per_warp, sbn.wpc, sbn.prog_words, s));
        ++b->launches;
      }
      for (const Bin& bin : b->dense_bins) {
        const int32_t* wl = part(bin, cnt);
        if (!cnt || bin.never) continue;
        KD_CK(launch_dense(v, sp, wl, cnt, bin.cap, bin.nt, false, s));
        ++b->launches;
        if (b->cl_smem && bin.nt == 256) {  // K2c: the PADMM of the bin's K2c worlds
          KD_CK(launch_dense_cluster(v, sp, wl, cnt, b->cl_smem, s));
          ++b->launches;
        }
      }
      {
        const int32_t* wl = part(b->global_bin, cnt);
        if (cnt && !b->global_bin.never) {
          if (b->global_bin.rare || b->slab_sweep_forced)
            KD_CK(launch_dense_global_sweep(v, sp, wl, cnt, b->global_bin.cap, s));
          else KD_CK(launch_dense(v, sp, wl, cnt, b->global_bin.cap, 256, true, s));
          ++b->launches;
        }
      }
    }
    mark(2);
    const Bin& cr = c->backend == KD_BACKEND_MATRIX_FREE ? b->cr_all_bin : b->cr_auto_bin;
    if (c->backend != KD_BACKEND_DENSE) {
      const int32_t* wl = part(cr, cnt);
      if (cnt) {
        KD_CK(launch_cr(v, sp, wl, cnt, cr.cap, cr.nbcap, cr.nt, s));
        ++b->launches;
      }
    }
    mark(3);
    launch_recover(v, sp, s, w0, w1);
    KD_CK(cudaGetLastError());
    ++b->launches;
    mark(4);
  }
  for (int p = 1; p < b->n_halves; ++p) {  // join: the main stream waits for every part
    KD_CK(cudaEventRecord(b->ev_join[p], b->pstream[p]));
    KD_CK(cudaStreamWaitEvent(b->stream, b->ev_join[p], 0));
  }
  if (b->timing) b->ev_used += 5 * (size_t)b->n_halves;  // per-family device time, resolved lazily
  return KD_OK;
}

// Nesterov coefficients (nesterov_next_coefficient / nesterov_update,
// padmm.cpp:54-71): a_0 = 1, a_{m+1} = (1 + sqrt(1 + 4 a_m^2)) / 2 and
// beta_m = (a_m - 1) / a_{m+1}.  The sequence restarts from a_0, so a PADMM
// loop only needs m (updates since the last restart); the host computes the
// table once in IEEE double, as the reference does.
static int ensure_nest_table(kd_batch* b, int max_iters) {
  if (max_iters <= b->nest_cap) return KD_OK;
  const int cap = std::max(256, max_iters);
  std::vector<double> t(cap);
  double a = 1.0;
  for (int m = 0; m < cap; ++m) {
    volatile double q = 4.0 * a * a;  // rounded product, never fused into the sum
    const double a_next = 0.5 * (1.0 + std::sqrt(1.0 + q));
    t[m] = (a - 1.0) / a_next;
    a = a_next;
  }
  double* d = nullptr;
  KD_CK(b->mem.alloc(d, cap));
  KD_CK(to_dev(b, d, t.data(), 8 * (size_t)cap));
  b->d_nest = d;
  b->nest_cap = cap;
  return KD_OK;
}

// backend = Dense: grow the dense-global slab to every world's full row
// capacity (once; Auto keeps using the same slab, whose worlds then have room
// for any n <= capacity).
static int ensure_dense_full(kd_batch* b) {
  if (b->dense_full || !b->has_big) return KD_OK;
  int64_t total = 0;
  std::vector<DevWorld> W = b->worlds;
  int cap = 0;
  for (int w : b->global_bin.worlds) {
    const int rcw = (int)((w + 1 < b->n_worlds ? b->row_off[w + 1] : b->total_rows) - b->row_off[w]);  // capacity
    W[w].slab_cap = rcw;
    W[w].lslab_off = total;
    total += slab_doubles(rcw);
    cap = std::max(cap, rcw);
  }
  double* slab = nullptr;
  if (cudaMalloc(&slab, 8 * (size_t)std::max<int64_t>(1, total)) != cudaSuccess) {
    cudaGetLastError();
    return fail(KD_ERR_CAPACITY, "dense backend: the factor storage of the worlds above 300 rows (" +
                                     std::to_string(8.0 * total / 1e9) + " GB) does not fit device memory");
  }
  KD_CK(cudaMemsetAsync(slab, 0, 8 * (size_t)std::max<int64_t>(1, total), b->stream));
  KD_CK(cudaStreamSynchronize(b->stream));
  b->mem.ptrs.push_back(slab);
  b->mem.release(b->view.lslab);
  b->view.lslab = slab;
  b->total_lslab = total;
  b->worlds = W;
  KD_CK(cudaMemcpyAsync(const_cast<DevWorld*>(b->view.worlds), W.data(), sizeof(DevWorld) * W.size(),
                        cudaMemcpyHostToDevice, b->stream));
  KD_CK(cudaStreamSynchronize(b->stream));
  b->global_bin.cap = cap;
  b->dense_full = true;
  b->drop_graph();
  return KD_OK;
}

static int enqueue_steps(kd_batch* b, const kd_step_config* c, int32_t n_steps) {
  const int nrc = ensure_nest_table(b, c->max_iters);
  if (nrc != KD_OK) return nrc;
  if (c->backend == KD_BACKEND_DENSE) {
    const int drc = ensure_dense_full(b);
    if (drc != KD_OK) return drc;
  }
  const StepParams sp = step_params(b, c);
  if (!b->graphs || b->timing || n_steps < 2) {
    for (int k = 0; k < n_steps; ++k) {
      const int rc = enqueue_one(b, c, sp);
      if (rc != KD_OK) return rc;
    }
    return KD_OK;
  }
  if (!b->graph_exec || std::memcmp(&b->graph_sp, &sp, sizeof(sp)) != 0 || b->graph_backend != c->backend) {
    b->drop_graph();
    const int64_t l0 = b->launches;
    int rc = enqueue_one(b, c, sp);  // direct first step (also sets the kernels' smem attributes)
    if (rc != KD_OK) return rc;
    --n_steps;
    const int64_t l1 = b->launches;
    KD_CK(cudaStreamBeginCapture(b->stream, cudaStreamCaptureModeThreadLocal));
    rc = enqueue_one(b, c, sp);
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(b->stream, &g);
    if (rc != KD_OK) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    KD_CK(e);
    b->graph = g;
    KD_CK(cudaGraphInstantiate(&b->graph_exec, g, 0));
    b->launches = l1;  // the captured step has not run yet
    b->graph_launches = (int)(l1 - l0);
    b->graph_sp = sp;
    b->graph_backend = c->backend;
  }
  for (int k = 0; k < n_steps; ++k) {
    KD_CK(cudaGraphLaunch(b->graph_exec, b->stream));
    b->launches += b->graph_launches;
  }
  return KD_OK;
}

int kd_batch_sync(kd_batch* b) {
  if (!b) return fail(KD_ERR_INVALID_ARGUMENT, "null batch");
  KD_CK(cudaSetDevice(b->device));
  KD_CK(cudaStreamSynchronize(b->stream));
  {
    const int rc = resolve_timing(b);
    if (rc != KD_OK) return rc;
  }
  int32_t err[4];
  KD_CK(to_host(b, err, b->d_err, 16));
  if (err[0]) return fail(KD_ERR_SPD_FAILURE, "Delassus factorization failed on an SPD system (" +
                                                  std::to_string(err[0]) + " worlds)");
  if (err[1]) return fail(KD_ERR_CAPACITY, "contact or dense-slab capacity exceeded in " + std::to_string(err[1]) +
                                               " worlds");
  return KD_OK;
}

int kd_batch_step_async(kd_batch* b, const kd_step_config* c, int32_t n_steps) {
  if (!b || !c) return fail(KD_ERR_INVALID_ARGUMENT, "null argument");
  if (b->n_worlds == 0 || n_steps <= 0) return KD_OK;
  KD_CK(cudaSetDevice(b->device));
  // the error word covers the steps of this call only (kd_batch_sync reads it)
  KD_CK(cudaMemsetAsync(b->d_err, 0, 16, b->stream));
  return enqueue_steps(b, c, n_steps);
}

int kd_batch_step(kd_batch* b, const kd_step_config* c, int32_t n_steps) {
  if (!b || !c) return fail(KD_ERR_INVALID_ARGUMENT, "null argument");
  if (b->n_worlds == 0 || n_steps <= 0) return KD_OK;
  KD_CK(cudaSetDevice(b->device));
  KD_CK(cudaMemsetAsync(b->d_err, 0, 16, b->stream));
  const int rc = enqueue_steps(b, c, n_steps);
  if (rc != KD_OK) return rc;
  return kd_batch_sync(b);
}

int kd_batch_assemble(kd_batch* b, const kd_step_config* c) {
  if (!b || !c) return fail(KD_ERR_INVALID_ARGUMENT, "null argument");
  if (b->n_worlds == 0) return KD_OK;
  KD_CK(cudaSetDevice(b->device));
  const int nrc = ensure_nest_table(b, c->max_iters);
  if (nrc != KD_OK) return nrc;
  const StepParams sp = step_params(b, c);
  KD_CK(cudaMemsetAsync(b->d_err, 0, 16, b->stream));
  launch_assemble(b->view, sp, b->stream);
  KD_CK(cudaGetLastError());
  KD_CK(cudaStreamSynchronize(b->stream));
  return KD_OK;
}

int kd_batch_stream(kd_batch* b, void** stream) {
  if (!b || !stream) return fail(KD_ERR_INVALID_ARGUMENT, "null argument");
  *stream = (void*)b->stream;
  return KD_OK;
}

int kd_batch_device_state(kd_batch* b, double** poses, double** twists, double** time) {
  if (!b) return fail(KD_ERR_INVALID_ARGUMENT, "null batch");
  if (poses) *poses = b->view.poses;
  if (twists) *twists = b->view.twists;
  if (time) *time = b->view.time;
  return KD_OK;
}

int kd_batch_fk(kd_batch* b, const int32_t* joints, const double* values, int32_t nt, double tol, int32_t max_iters,
                double lm0, int32_t* iterations, double* residual_inf, uint8_t* converged) {
  if (!b || nt < 0 || (nt > 0 && (!joints || !values))) return fail(KD_ERR_INVALID_ARGUMENT, "invalid arguments");
  if (b->n_worlds == 0) return KD_OK;
  KD_CK(cudaSetDevice(b->device));
  size_t smem = 0;
  for (int w = 0; w < b->n_worlds; ++w) {
    const HostModel& m = b->models[b->world_model[w]];
    for (int k = 0; k < nt; ++k) {
      const int j = joints[(size_t)w * nt + k];
      if (j < 0 || j >= (int)m.joints.size()) return fail(KD_ERR_INVALID_ARGUMENT, "target joint index out of range");
      const int t = m.joints[j].type;
      if (t != J_REVOLUTE && t != J_PRISMATIC)
        return fail(KD_ERR_MODEL_WRONG_JOINT_TYPE, "joint '" + m.joint_names[j] + "' has no scalar coordinate");
    }
    smem = std::max(smem, fk_smem_bytes((int)m.bodies.size(), m.n_bil + nt));
  }
  // models too large for one CTA's shared memory: a per-world HBM scratch slab
  double* d_scr = nullptr;
  if (smem > 232448) {
    const size_t per = (smem + 15) / 16 * 16;
    if (cudaMalloc(&d_scr, per * (size_t)b->n_worlds) != cudaSuccess) {
      cudaGetLastError();
      return fail(KD_ERR_CAPACITY, "forward kinematics: the normal-matrix scratch (" +
                                       std::to_string(per * (double)b->n_worlds / 1e9) + " GB) does not fit device memory");
    }
  }
  const size_t n = (size_t)b->n_worlds * std::max(1, nt);
  int32_t* d_j = nullptr;
  double* d_v = nullptr;
  int32_t* d_it = nullptr;
  double* d_res = nullptr;
  uint8_t* d_conv = nullptr;
  KD_CK(cudaMalloc(&d_j, 4 * n));
  KD_CK(cudaMalloc(&d_v, 8 * n));
  KD_CK(cudaMalloc(&d_it, 4 * (size_t)b->n_worlds));
  KD_CK(cudaMalloc(&d_res, 8 * (size_t)b->n_worlds));
  KD_CK(cudaMalloc(&d_conv, (size_t)b->n_worlds));
  int rc = KD_OK;
  if (nt > 0) {
    KD_CK(cudaMemcpyAsync(d_j, joints, 4 * (size_t)b->n_worlds * nt, cudaMemcpyHostToDevice, b->stream));
    KD_CK(cudaMemcpyAsync(d_v, values, 8 * (size_t)b->n_worlds * nt, cudaMemcpyHostToDevice, b->stream));
  }
  cudaError_t e = launch_fk(b->view, d_j, d_v, nt, tol, max_iters, lm0, d_it, d_res, d_conv, smem, b->stream, d_scr);
  if (e == cudaSuccess) e = cudaStreamSynchronize(b->stream);
  if (e == cudaSuccess && iterations) e = to_host(b, iterations, d_it, 4 * (size_t)b->n_worlds);
  if (e == cudaSuccess && residual_inf)
    e = to_host(b, residual_inf, d_res, 8 * (size_t)b->n_worlds);
  if (e == cudaSuccess && converged) e = to_host(b, converged, d_conv, (size_t)b->n_worlds);
  if (e != cudaSuccess) rc = fail(KD_ERR_CUDA, std::string("kd_batch_fk: ") + cudaGetErrorString(e));
  cudaFree(d_j);
  cudaFree(d_v);
  cudaFree(d_it);
  cudaFree(d_res);
  cudaFree(d_conv);
  if (d_scr) cudaFree(d_scr);
  return rc;
}

int kd_batch_set_state_async(kd_batch* b, const double* poses, const double* twists) {
  if (!b) return fail(KD_ERR_INVALID_ARGUMENT, "null batch");
  KD_CK(cudaSetDevice(b->device));
  if (poses && b->pose_len)
    KD_CK(cudaMemcpyAsync(b->view.poses, poses, 8 * b->pose_len, cudaMemcpyHostToDevice, b->stream));
  if (twists && b->twist_len)
    KD_CK(cudaMemcpyAsync(b->view.twists, twists, 8 * b->twist_len, cudaMemcpyHostToDevice, b->stream));
  return KD_OK;
}

int kd_batch_get_state_async(kd_batch* b, double* poses, double* twists) {
  if (!b) return fail(KD_ERR_INVALID_ARGUMENT, "null batch");
  KD_CK(cudaSetDevice(b->device));
  if (poses && b->pose_len)
    KD_CK(cudaMemcpyAsync(poses, b->view.poses, 8 * b->pose_len, cudaMemcpyDeviceToHost, b->stream));
  if (twists && b->twist_len)
    KD_CK(cudaMemcpyAsync(twists, b->view.twists, 8 * b->twist_len, cudaMemcpyDeviceToHost, b->stream));
  return KD_OK;
}

int kd_batch_get_diagnostics(kd_batch* b, kd_step_diag* out) {
  if (!b || !out) return fail(KD_ERR_INVALID_ARGUMENT, "null argument");
  KD_CK(cudaSetDevice(b->device));
  std::vector<WorldStep> ws(b->n_worlds);
  if (b->n_worlds)
    KD_CK(to_host(b, ws.data(), b->view.wstep, sizeof(WorldStep) * b->n_worlds));
  for (int w = 0; w < b->n_worlds; ++w) {
    const WorldStep& s = ws[w];
    const HostModel& m = b->models[b->world_model[w]];
    kd_step_diag& o = out[w];
    std::memset(&o, 0, sizeof(o));
    o.iterations = s.iterations;
    o.restarts = s.restarts;
    o.converged = s.converged;
    o.cr_breakdown = s.cr_breakdown;
    o.cr_iterations = s.cr_iterations;
    o.r_p = s.r_p;
    o.r_d = s.r_d;
    o.r_c = s.r_c;
    o.n_rows = std::max(0, s.n_rows);
    o.contact_count = s.n_contacts;
    o.first_contact_row = m.n_bil + m.n_dyn + s.n_limits;
    o.n_limits = s.n_limits;
    o.f_inf = s.f_inf;
    o.kkt_momentum_inf = s.kkt;
    o.bilateral_velocity_inf = s.bil_vel;
  }
  return KD_OK;
}

int kd_batch_get_phase_cycles(kd_batch* b, int64_t* out) {
  if (!b || !out) return fail(KD_ERR_INVALID_ARGUMENT, "null argument");
  KD_CK(cudaSetDevice(b->device));
  std::vector<WorldStep> ws(b->n_worlds);
  if (b->n_worlds)
    KD_CK(to_host(b, ws.data(), b->view.wstep, sizeof(WorldStep) * b->n_worlds));
  for (int w = 0; w < b->n_worlds; ++w)
    for (int k = 0; k < 8; ++k) out[8 * w + k] = (ws[w].backend == BE_DENSE_SMEM || ws[w].backend == BE_SPARSE || ws[w].backend == BE_DENSE_SN || ws[w].backend == BE_MATRIX_FREE) ? ws[w].phase_cycles[k] : 0;
  return KD_OK;
}

int kd_batch_get_kernels(kd_batch* b, int32_t* out) {
  if (!b || !out) return fail(KD_ERR_INVALID_ARGUMENT, "null argument");
  KD_CK(cudaSetDevice(b->device));
  std::vector<WorldStep> ws(b->n_worlds);
  if (b->n_worlds)
    KD_CK(to_host(b, ws.data(), b->view.wstep, sizeof(WorldStep) * b->n_worlds));
  for (int w = 0; w < b->n_worlds; ++w) {
    const int be = ws[w].backend;
    out[w] = be == BE_SPARSE ? KD_KERNEL_SUPERNODAL
             : (be == BE_DENSE_SMEM || be == BE_DENSE_GLOBAL) ? KD_KERNEL_DENSE
             : be == BE_DENSE_SN ? (b->worlds[w].xslab_off >= 0 ? KD_KERNEL_SUPERNODAL_CLUSTER : KD_KERNEL_SUPERNODAL_DENSE)
             : be == BE_MATRIX_FREE ? KD_KERNEL_CR : KD_KERNEL_NONE;
  }
  return KD_OK;
}

int kd_batch_get_cr_paths(kd_batch* b, int32_t* out) {
  if (!b || !out) return fail(KD_ERR_INVALID_ARGUMENT, "null argument");
  KD_CK(cudaSetDevice(b->device));
  std::vector<WorldStep> ws(b->n_worlds);
  if (b->n_worlds)
    KD_CK(to_host(b, ws.data(), b->view.wstep, sizeof(WorldStep) * b->n_worlds));
  for (int w = 0; w < b->n_worlds; ++w)
    out[w] = ws[w].backend == BE_MATRIX_FREE ? ws[w].cr_path : KD_CR_PATH_NONE;
  return KD_OK;
}

int kd_batch_row_offsets(const kd_batch* b, int64_t* ro, int64_t* total) {
  if (!b) return fail(KD_ERR_INVALID_ARGUMENT, "null batch");
  for (int w = 0; w < b->n_worlds; ++w) ro[w] = b->row_off[w];
  if (total) *total = b->total_rows;
  return KD_OK;
}

int kd_batch_get_impulses(kd_batch* b, double* out) {
  if (!b || !out) return fail(KD_ERR_INVALID_ARGUMENT, "null argument");
  KD_CK(cudaSetDevice(b->device));
  KD_CK(to_host(b, out, b->view.imp, 8 * b->total_rows));
  return KD_OK;
}

int kd_batch_dump_rows(kd_batch* b, int32_t w, kd_row_dump* out, int32_t cap, int32_t* n_rows) {
  if (!b || !out || !n_rows || w < 0 || w >= b->n_worlds) return fail(KD_ERR_INVALID_ARGUMENT, "invalid argument");
  KD_CK(cudaSetDevice(b->device));
  WorldStep s;
  KD_CK(to_host(b, &s, b->view.wstep + w, sizeof(s)));
  const int n = std::max(0, s.n_rows);
  *n_rows = n;
  if (n > cap) return fail(KD_ERR_CAPACITY, "dump capacity too small");
  if (n == 0) return KD_OK;
  const int64_t R0 = b->row_off[w];
  std::vector<RowJ> rj(n);
  std::vector<int32_t> rb(2 * n), rk(n);
  std::vector<double> bias(n), reg(n), scale(n), vf(n), lam(n), zo(n);
  const BatchView& v = b->view;
  KD_CK(to_host(b, rj.data(), v.rowj + R0, sizeof(RowJ) * n));
  KD_CK(to_host(b, rb.data(), v.rbody + 2 * R0, 8 * n));
  KD_CK(to_host(b, rk.data(), v.rkind + R0, 4 * n));
  KD_CK(to_host(b, bias.data(), v.bias + R0, 8 * n));
  KD_CK(to_host(b, reg.data(), v.reg + R0, 8 * n));
  KD_CK(to_host(b, scale.data(), v.scale + R0, 8 * n));
  KD_CK(to_host(b, vf.data(), v.vf + R0, 8 * n));
  KD_CK(to_host(b, lam.data(), v.lam + R0, 8 * n));
  KD_CK(to_host(b, zo.data(), v.zo + R0, 8 * n));
  for (int r = 0; r < n; ++r) {
    kd_row_dump& o = out[r];
    std::memset(&o, 0, sizeof(o));
    o.body_a = rb[2 * r];
    o.body_b = rb[2 * r + 1];
    o.kind = rk[r];
    for (int k = 0; k < 6; ++k) {
      o.block_a[k] = rj[r].J[k];
      o.block_b[k] = rj[r].J[6 + k];
    }
    o.bias = bias[r];
    o.reg = reg[r];
    o.scale = scale[r];
    o.vf_scaled = vf[r];
    o.lambda = lam[r];
    o.z = zo[r];
  }
  return KD_OK;
}

int kd_batch_dump_contacts(kd_batch* b, int32_t w, int32_t* geoms, double* data9, int32_t cap, int32_t* nc) {
  if (!b || !nc || w < 0 || w >= b->n_worlds) return fail(KD_ERR_INVALID_ARGUMENT, "invalid argument");
  KD_CK(cudaSetDevice(b->device));
  WorldStep s;
  KD_CK(to_host(b, &s, b->view.wstep + w, sizeof(s)));
  *nc = std::max(0, s.n_contacts);
  if (*nc > cap) return fail(KD_ERR_CAPACITY, "dump capacity too small");
  std::vector<Contact> ct(*nc);
  if (*nc)
    KD_CK(to_host(b, ct.data(), b->view.contacts + b->worlds[w].contact_off, sizeof(Contact) * *nc));
  for (int c = 0; c < *nc; ++c) {
    geoms[2 * c] = ct[c].ga;
    geoms[2 * c + 1] = ct[c].gb;
    double* d = data9 + 9 * c;
    for (int k = 0; k < 3; ++k) {
      d[k] = ct[c].pos[k];
      d[3 + k] = ct[c].nrm[k];
    }
    d[6] = ct[c].depth;
    d[7] = ct[c].mu;
    d[8] = ct[c].e;
  }
  return KD_OK;
}

int kd_batch_dump_limits(kd_batch* b, int32_t w, int32_t* keys2, int32_t cap, int32_t* nl) {
  if (!b || !nl || w < 0 || w >= b->n_worlds) return fail(KD_ERR_INVALID_ARGUMENT, "invalid argument");
  KD_CK(cudaSetDevice(b->device));
  WorldStep s;
  KD_CK(to_host(b, &s, b->view.wstep + w, sizeof(s)));
  *nl = std::max(0, s.n_limits);
  if (*nl > cap) return fail(KD_ERR_CAPACITY, "dump capacity too small");
  const HostModel& m = b->models[b->world_model[w]];
  const int64_t first = b->row_off[w] + m.n_bil + m.n_dyn;
  if (*nl) KD_CK(to_host(b, keys2, b->view.lkey + 2 * first, 8 * *nl));
  return KD_OK;
}

// ---- warm-start caches (extract_state / insert_state, batch.cpp:27-72)
int kd_batch_get_cache_sizes(kd_batch* b, int32_t w, int32_t* jl, int32_t* jv, int32_t* nl, int32_t* nc) {
  if (!b || w < 0 || w >= b->n_worlds) return fail(KD_ERR_INVALID_ARGUMENT, "invalid argument");
  KD_CK(cudaSetDevice(b->device));
  const HostModel& m = b->models[b->world_model[w]];
  const DevWorld& W = b->worlds[w];
  WorldStep s;
  KD_CK(to_host(b, &s, b->view.wstep + w, sizeof(s)));
  if (jl) *jl = m.n_bil + m.n_dyn;
  if (jv) *jv = s.jcache_valid;
  if (nl) {
    std::vector<int32_t> valid(2 * (size_t)m.info.n_limited_joints);
    if (!valid.empty()) KD_CK(to_host(b, valid.data(), b->view.ls_valid + W.lslot_off, 4 * valid.size()));
    int k = 0;
    for (int32_t v : valid) k += v != 0;
    *nl = k;
  }
  if (nc) *nc = s.ccache_count;
  return KD_OK;
}

int kd_batch_get_caches(kd_batch* b, int32_t w, double* jlam, double* jz, int32_t* jvalid, kd_limit_cache_entry* lim,
                        int32_t lcap, int32_t* nl, kd_contact_cache_entry* con, int32_t ccap, int32_t* nc) {
  if (!b || w < 0 || w >= b->n_worlds) return fail(KD_ERR_INVALID_ARGUMENT, "invalid argument");
  KD_CK(cudaSetDevice(b->device));
  const HostModel& m = b->models[b->world_model[w]];
  const DevWorld& W = b->worlds[w];
  const BatchView& v = b->view;
  WorldStep s;
  KD_CK(to_host(b, &s, v.wstep + w, sizeof(s)));
  const int njd = m.n_bil + m.n_dyn;
  if (jvalid) *jvalid = s.jcache_valid;
  if (jlam && njd) KD_CK(to_host(b, jlam, v.jc_lam + W.jcache_off, 8 * (size_t)njd));
  if (jz && njd) KD_CK(to_host(b, jz, v.jc_z + W.jcache_off, 8 * (size_t)njd));
  // limit slots 2 * limit_slot + bound, listed in (joint, bound) order
  const int nls = 2 * m.info.n_limited_joints;
  std::vector<int32_t> valid(nls);
  std::vector<double> ll(nls), lz(nls);
  if (nls) {
    KD_CK(to_host(b, valid.data(), v.ls_valid + W.lslot_off, 4 * (size_t)nls));
    KD_CK(to_host(b, ll.data(), v.ls_lam + W.lslot_off, 8 * (size_t)nls));
    KD_CK(to_host(b, lz.data(), v.ls_z + W.lslot_off, 8 * (size_t)nls));
  }
  int k = 0;
  for (size_t j = 0; j < m.joints.size(); ++j) {
    if (!(m.joints[j].flags & JF_LIMITS)) continue;
    for (int bound = 0; bound < 2; ++bound) {
      const int slot = 2 * m.joints[j].limit_slot + bound;
      if (!valid[slot]) continue;
      if (lim && k < lcap) lim[k] = kd_limit_cache_entry{(int32_t)j, bound, ll[slot], lz[slot]};
      ++k;
    }
  }
  if (nl) *nl = k;
  if (lim && k > lcap) return fail(KD_ERR_CAPACITY, "limit cache capacity too small");
  const int n = s.ccache_count;
  if (nc) *nc = n;
  if (con && n > ccap) return fail(KD_ERR_CAPACITY, "contact cache capacity too small");
  if (con && n) {
    std::vector<CacheEntry> ce(n);
    KD_CK(to_host(b, ce.data(), v.ccache + W.contact_off, sizeof(CacheEntry) * n));
    for (int c = 0; c < n; ++c) {
      kd_contact_cache_entry& o = con[c];
      o.geom_a = ce[c].ga;
      o.geom_b = ce[c].gb;
      for (int d = 0; d < 3; ++d) {
        o.position[d] = ce[c].pos[d];
        o.impulse[d] = ce[c].imp[d];
        o.dual[d] = ce[c].dual[d];
      }
    }
  }
  return KD_OK;
}

int kd_batch_set_caches(kd_batch* b, int32_t w, const double* jlam, const double* jz, int32_t jlen, int32_t jvalid,
                        const kd_limit_cache_entry* lim, int32_t nlim, const kd_contact_cache_entry* con,
                        int32_t ncon) {
  if (!b || w < 0 || w >= b->n_worlds || nlim < 0 || ncon < 0 || (nlim && !lim) || (ncon && !con))
    return fail(KD_ERR_INVALID_ARGUMENT, "invalid argument");
  KD_CK(cudaSetDevice(b->device));
  const HostModel& m = b->models[b->world_model[w]];
  const DevWorld& W = b->worlds[w];
  const BatchView& v = b->view;
  const int njd = m.n_bil + m.n_dyn;
  // contact entries -> model pair index (collide()'s pair list); the device
  // cache is kept sorted by pair (K1 bisects it).  A stable sort keeps the
  // entry order within a pair, the only order match_warmstart's (dist, entry,
  // contact) tie-break can see, since candidates compete only within a pair.
  std::vector<CacheEntry> ce;
  for (int c = 0; c < ncon; ++c) {
    int pair = -1;
    for (size_t p = 0; p < m.pairs.size() && pair < 0; ++p)
      if (m.pairs[p].a == con[c].geom_a && m.pairs[p].b == con[c].geom_b) pair = (int)p;
    if (pair < 0) continue;
    CacheEntry e{};
    e.ga = con[c].geom_a;
    e.gb = con[c].geom_b;
    e.pair = pair;
    for (int d = 0; d < 3; ++d) {
      e.pos[d] = con[c].position[d];
      e.imp[d] = con[c].impulse[d];
      e.dual[d] = con[c].dual[d];
    }
    ce.push_back(e);
  }
  std::stable_sort(ce.begin(), ce.end(), [](const CacheEntry& x, const CacheEntry& y) { return x.pair < y.pair; });
  if ((int)ce.size() > W.contact_cap)
    return fail(KD_ERR_CAPACITY, "contact cache: " + std::to_string(ce.size()) + " entries exceed the world's " +
                                     std::to_string(W.contact_cap) + "-contact capacity");
  WorldStep s;
  KD_CK(to_host(b, &s, v.wstep + w, sizeof(s)));
  s.jcache_valid = (jvalid && jlen == njd) ? 1 : 0;
  if (s.jcache_valid && njd) {
    if (!jlam || !jz) return fail(KD_ERR_INVALID_ARGUMENT, "joint cache arrays are null");
    KD_CK(to_dev(b, v.jc_lam + W.jcache_off, jlam, 8 * (size_t)njd));
    KD_CK(to_dev(b, v.jc_z + W.jcache_off, jz, 8 * (size_t)njd));
  }
  const int nls = 2 * m.info.n_limited_joints;
  if (nls) {
    std::vector<int32_t> valid(nls, 0);
    std::vector<double> ll(nls, 0.0), lz(nls, 0.0);
    for (int k = 0; k < nlim; ++k) {
      const int j = lim[k].joint, bound = lim[k].bound;
      if (j < 0 || j >= (int)m.joints.size() || bound < 0 || bound > 1 || !(m.joints[j].flags & JF_LIMITS)) continue;
      const int slot = 2 * m.joints[j].limit_slot + bound;
      valid[slot] = 1;
      ll[slot] = lim[k].lambda;
      lz[slot] = lim[k].z;
    }
    KD_CK(to_dev(b, v.ls_valid + W.lslot_off, valid.data(), 4 * (size_t)nls));
    KD_CK(to_dev(b, v.ls_lam + W.lslot_off, ll.data(), 8 * (size_t)nls));
    KD_CK(to_dev(b, v.ls_z + W.lslot_off, lz.data(), 8 * (size_t)nls));
  }
  if (!ce.empty()) KD_CK(to_dev(b, v.ccache + W.contact_off, ce.data(), sizeof(CacheEntry) * ce.size()));
  s.ccache_count = (int)ce.size();
  KD_CK(to_dev(b, v.wstep + w, &s, sizeof(s)));
  return KD_OK;
}

int kd_bench_jitter(uint64_t seed, double sigma, int32_t n_worlds, const int32_t* n_bodies, double* twists6) {
  if (!n_bodies || !twists6) return fail(KD_ERR_INVALID_ARGUMENT, "null argument");
  if (seed == 0) return KD_OK;  // main.cpp:204: jitter only for seed != 0
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> jitter(0.0, sigma);
  int64_t off = 0;
  for (int w = 0; w < n_worlds; ++w)
    for (int b = 0; b < n_bodies[w]; ++b, off += 6)
      for (int k = 0; k < 3; ++k) {
        twists6[off + k] += jitter(rng);
        twists6[off + 3 + k] += jitter(rng);
      }
  return KD_OK;
}

}  // extern "C"
