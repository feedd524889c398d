// Host runtime behind the C ABI (include/invaskit.h): problem upload in tree
// order, the level plan, and the factor / solve launch sequences.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <string>
#include <type_traits>
#include <atomic>
#include <thread>
#include <vector>

#include "../../include/invaskit.h"
#include "container.h"
#include "gemm.cuh"
#include "kernels.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define KS_CUDA(x)                                                                              \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess) return fail(KS_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #x,     \
                                       cudaGetErrorString(e_));                                 \
  } while (0)

constexpr double kCondHard = 1e14;  // solver.py:50
constexpr double kCondWarn = 1e10;  // solver.py:51

int64_t roundup(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

// Device memory for handles comes from the device's stream-ordered pool, which
// keeps up to KS_POOL_GB (default 32) GB of freed memory: a handle created
// after another one was destroyed (a new factorize call on the same shapes)
// reuses its memory instead of going back to the driver. Frees keep the
// device-wide synchronization cudaFree implies (buffers may still be in use on
// any of the handle's streams).
static cudaError_t pool_setup() {
  static int done = -1;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (done == dev) return cudaSuccess;
  cudaMemPool_t pool;
  if ((e = cudaDeviceGetDefaultMemPool(&pool, dev)) != cudaSuccess) return e;
  const char* env = std::getenv("KS_POOL_GB");
  uint64_t keep = (uint64_t)(env ? std::atof(env) : 32.0) << 30;
  if ((e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep)) != cudaSuccess) return e;
  done = dev;
  return cudaSuccess;
}

static cudaError_t pool_alloc(void** p, size_t bytes) {
  cudaError_t e = pool_setup();
  if (e != cudaSuccess) return e;
  if ((e = cudaMallocAsync(p, bytes, 0)) != cudaSuccess) return e;
  return cudaStreamSynchronize(0);  // usable from every stream once this returns
}

static void pool_free(void* p) {
  cudaDeviceSynchronize();
  cudaFreeAsync(p, 0);
  cudaStreamSynchronize(0);
}

template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaError_t alloc(size_t count) {
    n = count;
    if (count == 0) return cudaSuccess;
    return pool_alloc(reinterpret_cast<void**>(&p), count * sizeof(T));
  }
  cudaError_t upload(const std::vector<T>& v) {
    cudaError_t e = alloc(v.size());
    if (e != cudaSuccess || v.empty()) return e;
    return cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
  }
  void release() {
    if (p) pool_free(p);
    p = nullptr;
    n = 0;
  }
};

}  // namespace

struct ks_factor {
  int device = 0;
  int64_t n = 0, d = 0, n_nodes = 0;
  std::vector<int64_t> begin, end, left, right, rank, level;
  // plan
  std::vector<int> leaf_nodes;                 // leaf index -> node
  std::vector<std::vector<int>> levels;        // internal nodes per level, deepest first
  std::vector<int> level_first;                // internal index of each level's first node
  std::vector<int> int_nodes;                  // internal index -> node
  int n_int = 0;
  // subtree sharding (multi-GPU): this handle factors the subtree of shard_root
  // ("local" levels) and, after the level-k exchange, the levels above it ("top")
  int64_t shard_root = 0;
  int shard_level = 0;
  int n_local_levels = 0;
  // subtree pipelining: the deepest npipe levels split into kLeafChunks
  // subtrees, each factored on its own stream right after its own leaves
  // (children of a subtree's nodes lie in the same subtree one level down)
  int npipe = 0;
  int64_t loc_begin = 0, loc_end = 0;   // tree-order rows owned by the shard
  std::vector<int64_t> peers;           // nodes at the shard level (all shards' roots)
  bool local_factored = false;
  int m_pad = 0, s_pad = 0, t_pad = 0, T = 0, R = 0, pw = 32;
  // device tables
  DBuf<double> coords, xx;   // coords: n + m_pad rows (zero tail), tree order
  DBuf<int> rank_d, skel_pos;
  DBuf<int64_t> skel_off, coeff_off;
  DBuf<double> coeff;
  DBuf<int> leaf_node, leaf_begin, leaf_size, leaf_info;
  DBuf<int> int_node, int_left, int_right, int_info, piv, moves, pm;
  DBuf<double> lu_scratch;
  DBuf<unsigned> lu_sync;  // persistent-LU flags: 4 words per internal node + the watchdog word
  DBuf<double> dinv;  // condition estimator: diagonal-block inverses of every node's Z factors
  DBuf<double> lut;   // condition estimator: column-major copies of every node's Z factors (t_pad <= 512)
  DBuf<double> leafA, inv, hbuf, aug, bc, pn, norm1, cond;
  // solve scratch
  DBuf<double> z, c, tin, y, wtmp, bdev, xdev;
  DBuf<double> mv_c, mv_inc, mv_tot;
  int64_t mv_q = 0;
  int64_t q_cap = 0;
  double h = 1.0;
  double lam = 0.0;
  bool factored = false;
  cudaStream_t side = nullptr, cap = nullptr;
  // independent node groups run on their own streams so latency-bound kernels
  // (POTRF, LU panels, TRSM) of one group overlap the GEMMs of another
  static constexpr int kGroups = 8;  // stream slots; KS_GROUPS picks how many are used (default 8)
  cudaStream_t gst[kGroups] = {};
  cudaEvent_t gfork = nullptr, gjoin[kGroups] = {};
  cudaEvent_t ev_phase[5] = {};
  std::vector<cudaEvent_t> ev_level;
  cudaGraphExec_t graph_exec = nullptr;
  bool graph_profiling = false;
  int64_t graph_launches = 0;
  int64_t n_factorizations = 0;
  DBuf<double> lam_dev;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // narrow levels' condition estimates: their own stream, so they do not queue
  // behind the deferred wide-level batch on `side`
  cudaStream_t side2 = nullptr;
  cudaEvent_t ev_fork2 = nullptr, ev_join2 = nullptr;
  // uploads started by ks_create, consumed by the first factorization
  static constexpr int kLeafChunks = 8;
  cudaStream_t upl = nullptr;
  cudaEvent_t ev_up_coords = nullptr, ev_up_all = nullptr, ev_up_leaf[kLeafChunks] = {}, ev_up_sub[kLeafChunks] = {};
  std::vector<cudaEvent_t> ev_up_level;
  bool upload_pending = false;
  // diagnostics
  std::vector<int> leaf_info_h, int_info_h;
  std::vector<double> cond_h;
  std::vector<int64_t> fallback;
  // LU fallback leaves (non-SPD leaf blocks, solver.py:125-131)
  std::vector<int> fb_leaf;  // leaf indices
  int fb_T = 0;
  DBuf<double> fb_aug, fb_y, fb_norm1, fb_cond;
  DBuf<int> fb_piv, fb_info, fb_moves, fb_pm, fb_node, fb_begin, fb_size;
  int64_t fb_q = 0;
  ks::NodeBatch fb_batch() const {
    ks::NodeBatch nb{};
    nb.count = (int)fb_leaf.size();
    nb.first = 0;
    nb.node = fb_node.p;
    nb.left = fb_node.p;
    nb.right = fb_node.p;
    nb.s_pad = fb_T - m_pad;
    nb.t_pad = m_pad;
    nb.T = fb_T;
    nb.Aug = fb_aug.p;
    nb.Bc = nullptr;
    nb.Pn = nullptr;
    nb.piv = fb_piv.p;
    nb.norm1 = fb_norm1.p;
    nb.cond = fb_cond.p;
    nb.info = fb_info.p;
    nb.moves = fb_moves.p;
    nb.pm = fb_pm.p;
    nb.scratch = nullptr;
    return nb;
  }
  // profiling
  bool profiling = false;
  double phase_ms[6] = {0, 0, 0, 0, 0, 0};
  std::vector<double> level_ms;
  // KS_TRACE=1: an event after every launch on the main stream; consecutive
  // deltas are per-kernel device times (including launch gaps)
  std::vector<cudaEvent_t> trace_ev;
  std::vector<const char*> trace_name;
  std::vector<int> trace_tag;
  int cur_tag = -1;  // -1 leaves, else internal level index
  int trace_n = 0;
  std::string trace_report;
  int64_t launches[2] = {0, 0};

  ks::DevTree devtree() const {
    ks::DevTree t;
    t.n = n;
    t.d = d;
    t.coords = coords.p;
    t.rank = rank_d.p;
    t.skel_off = skel_off.p;
    t.skel_pos = skel_pos.p;
    t.coeff_off = coeff_off.p;
    t.coeff = coeff.p;
    t.h = h;
    return t;
  }
  ks::LeafBatch leafbatch() const {
    ks::LeafBatch lb;
    lb.count = (int)leaf_nodes.size();
    lb.node = leaf_node.p;
    lb.begin = leaf_begin.p;
    lb.size = leaf_size.p;
    lb.m_pad = m_pad;
    lb.s_pad = s_pad;
    lb.A = leafA.p;
    lb.a_stride = (int64_t)R * m_pad;
    return lb;
  }
  ks::NodeBatch nodebatch(int lev) const {
    const int first = level_first[lev];
    ks::NodeBatch nb;
    nb.count = (int)levels[lev].size();
    nb.first = first;
    nb.node = int_node.p + first;
    nb.left = int_left.p + first;
    nb.right = int_right.p + first;
    nb.s_pad = s_pad;
    nb.t_pad = t_pad;
    nb.T = T;
    nb.Aug = aug.p + (int64_t)first * T * T;
    nb.Bc = bc.p + (int64_t)first * s_pad * s_pad;
    nb.Pn = pn.p + (int64_t)first * s_pad * t_pad;
    nb.piv = piv.p + (int64_t)first * t_pad;
    nb.norm1 = norm1.p + first;
    nb.cond = cond.p + first;
    nb.info = int_info.p + first;
    nb.moves = moves.p + (int64_t)first * (2 * 64 + 1);
    nb.pm = pm.p + (int64_t)first * t_pad;
    nb.scratch = lu_scratch.p + (int64_t)first * 32 * 64;
    return nb;
  }
  void release_all() {
    coords.release(); xx.release(); rank_d.release(); skel_pos.release(); skel_off.release(); coeff_off.release();
    coeff.release(); leaf_node.release(); leaf_begin.release(); leaf_size.release(); leaf_info.release();
    int_node.release(); int_left.release(); int_right.release(); int_info.release(); piv.release(); moves.release(); pm.release(); lu_scratch.release(); lu_sync.release(); dinv.release(); lut.release();
    leafA.release(); inv.release(); hbuf.release(); aug.release(); bc.release(); pn.release();
    norm1.release(); cond.release(); z.release(); c.release(); tin.release(); y.release();
    fb_aug.release(); fb_y.release(); fb_norm1.release(); fb_cond.release(); fb_piv.release(); fb_info.release();
    fb_moves.release(); fb_pm.release(); fb_node.release(); fb_begin.release(); fb_size.release();
    wtmp.release(); bdev.release(); xdev.release(); mv_c.release(); mv_inc.release(); mv_tot.release();
  }
};

namespace {

using ks::GemmArgs;
using ks::Operand;
using ks::OperandW;

GemmArgs mk(int M, int N, int K, int batch, Operand A, Operand B, OperandW C, double alpha, double beta) {
  GemmArgs g;
  g.M = M; g.N = N; g.K = K; g.batch = batch;
  g.A = A; g.B = B; g.C = C;
  g.alpha = alpha; g.beta = beta; g.tri = 0;
  g.E = Operand{nullptr, 0, 0, nullptr};
  return g;
}

bool trace_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("KS_TRACE");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

bool debug_sync() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("KS_DEBUG_SYNC");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

struct Launcher {
  ks_factor* f;
  cudaStream_t st;
  int64_t* count;
  // KS_DEBUG_SYNC=1: synchronize after every launch so errors name their kernel
  int check(const char* what) {
    if (trace_on() && f) {
      if (f->trace_n >= (int)f->trace_ev.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        f->trace_ev.push_back(e);
        f->trace_name.push_back(what);
        f->trace_tag.push_back(-1);
      }
      f->trace_name[f->trace_n] = what;
      f->trace_tag[f->trace_n] = f->cur_tag;
      cudaEventRecord(f->trace_ev[f->trace_n++], st);
    }
    if (!debug_sync()) return KS_OK;
    cudaError_t e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return fail(KS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return KS_OK;
  }
  int gemm(const GemmArgs& g, bool ta, bool tb, const char* name = "gemm") {
    ++*count;
    cudaError_t e = ks::gemm(g, ta, tb, st);
    if (e != cudaSuccess) return fail(KS_ERR_CUDA, "gemm %dx%dx%d: %s", g.M, g.N, g.K, cudaGetErrorString(e));
    return check(name);
  }
};

// B[r0:r0+w, c0:c0+ncols] := L^-1 B, L unit lower at (r0, r0) of each node's Aug.
int trsm_ul(Launcher& L, const ks::NodeBatch& nb, int r0, int w, int c0, int ncols) {
  if (ncols <= 0) return KS_OK;
  if (w == 8 || w == 16 || w == 32 || w == 64) {
    ks::launch_trsm_unit_lower(nb, r0, w, c0, ncols, L.st);
    ++*L.count;
    return L.check("trsm_unit_lower");
  }
  // w is a multiple of 8; split into base sizes
  const int h = (w > 64) ? (int)roundup(w / 2, 8) : (w > 32 ? 32 : (w > 16 ? 16 : 8));
  int rc = trsm_ul(L, nb, r0, h, c0, ncols);
  if (rc) return rc;
  const int64_t TT = (int64_t)nb.T * nb.T;
  Operand A{nb.Aug + (int64_t)(r0 + h) * nb.T + r0, nb.T, TT, nullptr};
  Operand B{nb.Aug + (int64_t)r0 * nb.T + c0, nb.T, TT, nullptr};
  OperandW C{nb.Aug + (int64_t)(r0 + h) * nb.T + c0, nb.T, TT, nullptr};
  rc = L.gemm(mk(w - h, ncols, h, nb.count, A, B, C, -1.0, 1.0), false, false, "trsm_gemm");
  if (rc) return rc;
  return trsm_ul(L, nb, r0 + h, w - h, c0, ncols);
}

// The fused TRSM+update merge (k_lu_merge) is opt-in: measured slower than the
// separate trsm_ul + rlu_gemm launches at config 3 (90.3 vs 86.7 ms).
bool fused_merge_off() {
  const char* e = std::getenv("KS_FUSED_MERGE");
  return !(e && e[0] == '1');
}

// Recursive LU of columns [c0, c0+w) over rows [c0, T), pivots among rows < t_pad.
// ext > 0: the ext columns right after [c0, c0+w) (the P^T block, on the right
// spine of the recursion) take part in every merge as part of the right block,
// so U12 = L^-1 Pi P^T and the Schur block H come out of the merges' TRSMs and
// GEMMs instead of a separate TRSM chain and Schur GEMM after the LU.
int rlu(Launcher& L, const ks::NodeBatch& nb, int c0, int w, int pw, int* pend, int ext = 0) {
  const int64_t TT = (int64_t)nb.T * nb.T;
  if (w <= pw) {
    if (w == 32 && pend[2] == 0 && ks::lu_panel32_ok(nb))
      ks::launch_lu_panel32(nb, c0, L.st);  // two 16-column halves and their merge in one launch
    else
      ks::launch_lu_panel(nb, c0, w, L.st, pend);  // panel LU + its row interchanges everywhere else
    pend[2] = 0;                                   // the pending U12 block (if any) is in place now
    *L.count += 1;
    if (int rc = L.check("lu_panel")) return rc;
    if (ext <= 0) return KS_OK;
    int rc = trsm_ul(L, nb, c0, w, c0 + w, ext);
    if (rc) return rc;
    Operand A{nb.Aug + (int64_t)(c0 + w) * nb.T + c0, nb.T, TT, nullptr};
    Operand B{nb.Aug + (int64_t)c0 * nb.T + c0 + w, nb.T, TT, nullptr};
    OperandW C{nb.Aug + (int64_t)(c0 + w) * nb.T + c0 + w, nb.T, TT, nullptr};
    return L.gemm(mk(nb.T - c0 - w, ext, w, nb.count, A, B, C, -1.0, 1.0), false, false, "rlu_gemm");
  }
  const int h = (int)roundup(w / 2, pw);
  int rc = rlu(L, nb, c0, h, pw, pend);
  if (rc) return rc;
  if ((h == 16 || h == 32) && w - h <= 64 && ext == 0 && !fused_merge_off() && nb.scratch) {
    ks::launch_lu_merge(nb, c0, h, w, L.st);  // TRSM + trailing GEMM in one launch
    ++*L.count;
    if ((rc = L.check("lu_merge"))) return rc;
    pend[0] = c0; pend[1] = c0 + h; pend[2] = h; pend[3] = w - h;  // U12 -> next panel kernel
    return rlu(L, nb, c0 + h, w - h, pw, pend);
  }
  rc = trsm_ul(L, nb, c0, h, c0 + h, w - h + ext);
  if (rc) return rc;
  Operand A{nb.Aug + (int64_t)(c0 + h) * nb.T + c0, nb.T, TT, nullptr};
  Operand B{nb.Aug + (int64_t)c0 * nb.T + c0 + h, nb.T, TT, nullptr};
  OperandW C{nb.Aug + (int64_t)(c0 + h) * nb.T + c0 + h, nb.T, TT, nullptr};
  rc = L.gemm(mk(nb.T - c0 - h, w - h + ext, h, nb.count, A, B, C, -1.0, 1.0), false, false, "rlu_gemm");
  if (rc) return rc;
  return rlu(L, nb, c0 + h, w - h, pw, pend, ext);
}

struct PhaseTimer {
  bool on;
  cudaStream_t st;
  std::vector<cudaEvent_t> ev;
  PhaseTimer(bool on_, cudaStream_t s, int n) : on(on_), st(s) {
    if (!on) return;
    ev.resize(n);
    for (auto& e : ev) cudaEventCreate(&e);
  }
  void mark(int i) {
    if (on) cudaEventRecord(ev[i], st);
  }
  float between(int a, int b) {
    float ms = 0.f;
    if (on) cudaEventElapsedTime(&ms, ev[a], ev[b]);
    return ms;
  }
  ~PhaseTimer() {
    for (auto& e : ev) cudaEventDestroy(e);
  }
};

int ensure_solve_bufs(ks_factor* f, int64_t q) {
  if (q <= f->q_cap) return KS_OK;
  f->z.release(); f->c.release(); f->tin.release(); f->y.release(); f->wtmp.release(); f->bdev.release();
  f->xdev.release();
  KS_CUDA(f->z.alloc((size_t)f->leaf_nodes.size() * f->m_pad * q));
  KS_CUDA(f->c.alloc((size_t)std::max<int64_t>(f->n_nodes * f->s_pad * q, 1)));
  KS_CUDA(f->tin.alloc((size_t)std::max<int64_t>(f->n_nodes * f->s_pad * q, 1)));
  KS_CUDA(f->y.alloc((size_t)std::max<int64_t>((int64_t)f->n_int * f->t_pad * q, 1)));
  KS_CUDA(f->wtmp.alloc((size_t)std::max<int64_t>((int64_t)f->n_int * f->t_pad * q, 1)));
  KS_CUDA(f->bdev.alloc((size_t)f->n * q));
  KS_CUDA(f->xdev.alloc((size_t)f->n * q));
  f->q_cap = q;
  return KS_OK;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace

extern "C" {

int ks_last_error(char* buf, int64_t len) {
  if (!buf || len <= 0) return (int)g_err.size();
  std::snprintf(buf, (size_t)len, "%s", g_err.c_str());
  return (int)g_err.size();
}

const char* ks_version(void) { return "libinvaskit 0.1 sm_100a (DMMA fp64, telescoping solve)"; }

static double host_ms() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

static bool host_timing() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("KS_HOST_TIMING");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// subtree pipelining covers the deepest levels with at least KS_PIPE_MIN
// (default 16) nodes per subtree
static int pipe_min_nodes() {
  const char* e = std::getenv("KS_PIPE_MIN");
  return e ? std::max(1, std::atoi(e)) : 16;
}

static int create_impl(const ks_problem* p, int device, int64_t shard_root, ks_factor** out) {
  const double t_start = host_ms();
  if (!p || !out) return fail(KS_ERR_INVALID, "null argument");
  *out = nullptr;
  if (p->n < 1 || p->d < 1 || p->n_nodes < 1) return fail(KS_ERR_INVALID, "empty problem");
  if (!(p->bandwidth > 0.0) || !std::isfinite(p->bandwidth))
    return fail(KS_ERR_INVALID, "gaussian kernel needs bandwidth > 0, got %g", p->bandwidth);
  KS_CUDA(cudaSetDevice(device));
  ks_factor* f = new ks_factor();
  f->device = device;
  f->n = p->n;
  f->d = p->d;
  f->n_nodes = p->n_nodes;
  f->h = p->bandwidth;
  const int64_t nn = p->n_nodes;
  f->begin.assign(p->node_begin, p->node_begin + nn);
  f->end.assign(p->node_end, p->node_end + nn);
  f->left.assign(p->node_left, p->node_left + nn);
  f->right.assign(p->node_right, p->node_right + nn);
  f->rank.assign(p->rank, p->rank + nn);
  auto bad = [&](const char* msg) {
    delete f;
    return fail(KS_ERR_INVALID, "%s", msg);
  };
  // levels by BFS from the root; validate the node table (tree.py:98-127)
  f->level.assign(nn, -1);
  f->level[0] = 0;
  if (f->begin[0] != 0 || f->end[0] != p->n) return bad("root must own [0, n)");
  std::vector<int> order{0};
  for (size_t i = 0; i < order.size(); ++i) {
    const int v = order[i];
    if (f->left[v] < 0) {
      if (f->right[v] >= 0) return bad("node with one child");
      continue;
    }
    const int64_t l = f->left[v], r = f->right[v];
    if (l <= 0 || r <= 0 || l >= nn || r >= nn || f->level[l] >= 0 || f->level[r] >= 0) return bad("bad child ids");
    if (f->begin[l] != f->begin[v] || f->end[l] != f->begin[r] || f->end[r] != f->end[v]) return bad("children do not split the parent range");
    f->level[l] = f->level[r] = f->level[v] + 1;
    order.push_back((int)l);
    order.push_back((int)r);
  }
  if ((int64_t)order.size() != nn) return bad("unreachable nodes in the tree");
  int depth = 0;
  int64_t m_max = 0, s_max = 0;
  for (int64_t v = 0; v < nn; ++v) {
    depth = std::max<int>(depth, (int)f->level[v] + 1);
    if (f->left[v] < 0) {
      f->leaf_nodes.push_back((int)v);
      m_max = std::max(m_max, f->end[v] - f->begin[v]);
      if (f->end[v] <= f->begin[v]) return bad("empty leaf");
    }
    if (f->rank[v] < 0) return bad("negative rank");
    s_max = std::max(s_max, f->rank[v]);
    const bool root = (v == 0);
    if (!root && f->rank[v] < 1) return bad("non-root node without a skeleton");
    if (root && f->rank[v] != 0) return bad("the root has no skeleton");
    const int64_t cand = (f->left[v] < 0) ? (f->end[v] - f->begin[v]) : (f->rank[f->left[v]] + f->rank[f->right[v]]);
    if (p->skel_off[v + 1] - p->skel_off[v] != f->rank[v]) return bad("skel_off inconsistent with rank");
    if (p->coeff_off[v + 1] - p->coeff_off[v] != f->rank[v] * cand) return bad("coeff_off inconsistent with rank x |cand|");
  }
  if (shard_root < 0 || shard_root >= nn) return bad("shard root out of range");
  f->shard_root = shard_root;
  f->shard_level = (int)f->level[shard_root];
  f->loc_begin = f->begin[shard_root];
  f->loc_end = f->end[shard_root];
  std::vector<char> in_sub(nn, 0);
  {
    std::vector<int64_t> st{shard_root};
    while (!st.empty()) {
      const int64_t v = st.back();
      st.pop_back();
      in_sub[v] = 1;
      if (f->left[v] >= 0) { st.push_back(f->left[v]); st.push_back(f->right[v]); }
    }
  }
  for (int64_t v = 0; v < nn; ++v) {
    if (f->level[v] < f->shard_level && f->left[v] < 0)
      return bad("sharding needs every node above the shard level to be internal");
    if (f->level[v] == f->shard_level) f->peers.push_back(v);
  }
  f->leaf_nodes.clear();
  m_max = 0;
  for (int64_t v = 0; v < nn; ++v)
    if (in_sub[v] && f->left[v] < 0) {
      f->leaf_nodes.push_back((int)v);
      m_max = std::max(m_max, f->end[v] - f->begin[v]);
    }
  // internal levels: the shard's own (deepest first), then the top levels
  std::vector<std::vector<int>> loc(depth), top(depth);
  for (int64_t v = 0; v < nn; ++v) {
    if (f->left[v] < 0) continue;
    if (in_sub[v]) loc[f->level[v]].push_back((int)v);
    else if (f->level[v] < f->shard_level) top[f->level[v]].push_back((int)v);
  }
  for (int l = depth - 1; l >= 0; --l)
    if (!loc[l].empty()) f->levels.push_back(loc[l]);
  f->n_local_levels = (int)f->levels.size();
  for (int l = depth - 1; l >= 0; --l)
    if (!top[l].empty()) f->levels.push_back(top[l]);
  for (auto& lv : f->levels) {
    f->level_first.push_back((int)f->int_nodes.size());
    for (int v : lv) f->int_nodes.push_back(v);
  }
  f->n_int = (int)f->int_nodes.size();
  {  // subtree pipelining plan
    const int G = ks_factor::kLeafChunks;
    const size_t nlv = f->leaf_nodes.size();
    std::vector<int> grp(nn, -1);
    if (nlv % G == 0 && nlv >= (size_t)G)
      for (size_t li = 0; li < nlv; ++li) grp[f->leaf_nodes[li]] = (int)(li / (nlv / G));
    for (int lev = 0; lev < f->n_local_levels && nlv % G == 0; ++lev) {
      const auto& lv = f->levels[lev];
      const int c = (int)lv.size();
      if (c % G || c / G < pipe_min_nodes()) break;
      bool ok = true;
      for (int i = 0; i < c; ++i) {
        const int g = i / (c / G), v = lv[i];
        if (grp[f->left[v]] != g || grp[f->right[v]] != g) ok = false;
      }
      if (!ok) break;
      for (int i = 0; i < c; ++i) grp[lv[i]] = i / (c / G);
      f->npipe = lev + 1;
    }
  }
  f->m_pad = (int)roundup(m_max, 64);
  f->s_pad = (int)roundup(s_max, 64);
  f->t_pad = 2 * f->s_pad;
  f->T = 3 * f->s_pad;
  f->R = f->m_pad + f->s_pad;
  // LU panel width of the launch sequence: register panels of 16 columns (up to
  // 1024 candidate rows, 8 beyond). KS_PANEL_W=32 selects 32-column panels where
  // they fit in shared memory: two 16-column halves and their merge in one
  // launch (k_lu_panel32) -- measured slower at config 3 (69.6 vs 69.1 ms: the
  // merge then runs on one SM per node instead of a grid); 8 forces narrow panels.
  f->pw = (f->T <= 1024) ? 16 : 8;
  if (const char* e = std::getenv("KS_PANEL_W")) {
    const int w = std::atoi(e);
    ks::NodeBatch probe{};
    probe.t_pad = f->t_pad;
    probe.T = f->T;
    if (w == 32 && ks::lu_panel32_ok(probe)) f->pw = 32;
    else if (w == 8) f->pw = 8;
  }
  if (f->T > 2048) { delete f; return fail(KS_ERR_UNSUPPORTED, "skeleton rank %lld too large (max 682)", (long long)s_max); }

  const double t_plan = host_ms();
  // the permutation first: the device gather of the points trusts it. Host
  // worker threads (the inverse is N random writes): pass 1 range-checks and
  // inverts, pass 2 confirms pos[perm[i]] == i (any duplicate fails it).
  auto parallel_for = [](int64_t n, auto&& body) {
    const int nth = (int)std::max<int64_t>(1, std::min<int64_t>(16, n / (1 << 16)));
    std::vector<std::thread> th;
    for (int t = 1; t < nth; ++t) th.emplace_back([&, t]() { body(n * t / nth, n * (t + 1) / nth); });
    body(0, n / nth);
    for (auto& x : th) x.join();
  };
  std::vector<int64_t> pos(p->n);
  std::atomic<int> perm_bad{0};
  parallel_for(p->n, [&](int64_t a, int64_t b) {
    for (int64_t i = a; i < b; ++i) {
      const int64_t id = p->perm[i];
      if (id < 0 || id >= p->n) { perm_bad = 1; return; }
      pos[id] = i;
    }
  });
  if (!perm_bad)
    parallel_for(p->n, [&](int64_t a, int64_t b) {
      for (int64_t i = a; i < b; ++i)
        if (pos[p->perm[i]] != i) { perm_bad = 1; return; }
    });
  if (perm_bad) return bad("perm is not a permutation");
  const size_t nl = f->leaf_nodes.size();
  const int64_t nsk = p->skel_off[nn];
  std::vector<int> sp((size_t)nsk);
  std::atomic<int> skel_bad{0};
  parallel_for(nsk, [&](int64_t a, int64_t b) {
    for (int64_t i = a; i < b; ++i) {
      const int64_t id = p->skel[i];
      if (id < 0 || id >= p->n) { skel_bad = 1; return; }
      sp[i] = (int)pos[id];
    }
  });
  if (skel_bad) return bad("skeleton id out of range");
  std::vector<int64_t> so(p->skel_off, p->skel_off + nn + 1), co(p->coeff_off, p->coeff_off + nn + 1);
  std::vector<int> rk(nn);
  for (int64_t v = 0; v < nn; ++v) rk[v] = (int)f->rank[v];
  std::vector<int> ln, lbg, lsz;
  for (int v : f->leaf_nodes) {
    ln.push_back(v);
    lbg.push_back((int)f->begin[v]);
    lsz.push_back((int)(f->end[v] - f->begin[v]));
  }
  std::vector<int> inode, ileft, iright;
  for (int v : f->int_nodes) {
    inode.push_back(v);
    ileft.push_back((int)f->left[v]);
    iright.push_back((int)f->right[v]);
  }
  // From here on the handle owns device memory and streams: errors go through ks_destroy.
  auto abort_create = [&](int rc) {
    ks_destroy(f);
    return rc;
  };
  auto alloc_all = [&]() -> int {
    KS_CUDA(f->rank_d.alloc(rk.size()));
    KS_CUDA(f->skel_pos.alloc(sp.size()));
    KS_CUDA(f->skel_off.alloc(so.size()));
    KS_CUDA(f->coeff_off.alloc(co.size()));
    KS_CUDA(f->leaf_node.alloc(ln.size()));
    KS_CUDA(f->leaf_begin.alloc(lbg.size()));
    KS_CUDA(f->leaf_size.alloc(lsz.size()));
    KS_CUDA(f->leaf_info.alloc(nl));
    KS_CUDA(f->int_node.alloc(inode.size()));
    KS_CUDA(f->int_left.alloc(ileft.size()));
    KS_CUDA(f->int_right.alloc(iright.size()));
    KS_CUDA(f->int_info.alloc(std::max(f->n_int, 1)));
    KS_CUDA(f->lu_sync.alloc((size_t)4 * f->n_int + 1));
    KS_CUDA(f->piv.alloc((size_t)std::max(f->n_int, 1) * f->t_pad + 1));
    KS_CUDA(f->moves.alloc((size_t)std::max(f->n_int, 1) * (2 * 64 + 1)));
    KS_CUDA(f->pm.alloc((size_t)std::max(f->n_int, 1) * f->t_pad + 1));
    KS_CUDA(f->lu_scratch.alloc((size_t)std::max(f->n_int, 1) * 32 * 64));
    KS_CUDA(f->dinv.alloc((size_t)std::max(f->n_int, 1) * 2 * f->t_pad * 16));
    if (f->t_pad <= 512) KS_CUDA(f->lut.alloc((size_t)std::max(f->n_int, 1) * f->t_pad * f->t_pad));
    KS_CUDA(f->leafA.alloc(nl * (size_t)f->R * f->m_pad));
    KS_CUDA(f->inv.alloc(nl * (size_t)f->m_pad * 64));
    KS_CUDA(f->hbuf.alloc((size_t)nn * f->s_pad * f->s_pad + 1));
    KS_CUDA(f->aug.alloc((size_t)f->n_int * f->T * f->T + 1));
    KS_CUDA(f->bc.alloc((size_t)f->n_int * f->s_pad * f->s_pad + 1));
    KS_CUDA(f->pn.alloc((size_t)f->n_int * f->s_pad * f->t_pad + 1));
    KS_CUDA(f->norm1.alloc(std::max(f->n_int, 1)));
    KS_CUDA(f->cond.alloc(std::max(f->n_int, 1)));
    KS_CUDA(f->coords.alloc((size_t)(p->n + f->m_pad) * p->d));
    KS_CUDA(f->xx.alloc((size_t)p->n + f->m_pad));
    KS_CUDA(f->coeff.alloc((size_t)p->coeff_off[nn]));
    KS_CUDA(cudaStreamCreateWithFlags(&f->side, cudaStreamNonBlocking));
    KS_CUDA(cudaStreamCreateWithFlags(&f->side2, cudaStreamNonBlocking));
    KS_CUDA(cudaEventCreateWithFlags(&f->ev_fork2, cudaEventDisableTiming));
    KS_CUDA(cudaEventCreateWithFlags(&f->ev_join2, cudaEventDisableTiming));
    KS_CUDA(cudaStreamCreateWithFlags(&f->cap, cudaStreamNonBlocking));
    for (auto& g : f->gst) KS_CUDA(cudaStreamCreateWithFlags(&g, cudaStreamNonBlocking));
    KS_CUDA(cudaEventCreateWithFlags(&f->gfork, cudaEventDisableTiming));
    for (auto& e : f->gjoin) KS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : f->ev_phase) KS_CUDA(cudaEventCreate(&e));
    f->ev_level.resize(f->levels.size());
    for (auto& e : f->ev_level) KS_CUDA(cudaEventCreate(&e));
    KS_CUDA(f->lam_dev.alloc(1));
    KS_CUDA(cudaEventCreateWithFlags(&f->ev_fork, cudaEventDisableTiming));
    KS_CUDA(cudaEventCreateWithFlags(&f->ev_join, cudaEventDisableTiming));
    return KS_OK;
  };
  if (int rc = alloc_all()) return abort_create(rc);
  const double t_alloc = host_ms();
  // ---- asynchronous uploads on the upload stream, in the order the first
  // factorization consumes them; the point-coordinate check overlaps the DMA.
  // Points: tree order on the device (coords_tree[i] = coords[perm[i]]) + norms.
  auto start_uploads = [&]() -> int {
    KS_CUDA(cudaStreamCreateWithFlags(&f->upl, cudaStreamNonBlocking));
    KS_CUDA(cudaEventCreateWithFlags(&f->ev_up_coords, cudaEventDisableTiming));
    KS_CUDA(cudaEventCreateWithFlags(&f->ev_up_all, cudaEventDisableTiming));
    for (auto& e : f->ev_up_leaf) KS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : f->ev_up_sub) KS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    f->ev_up_level.resize(f->levels.size());
    for (auto& e : f->ev_up_level) KS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cudaStream_t u = f->upl;
    // the small tables first (pageable sources: staged before the call returns)
    auto put = [&](auto& buf, const auto& v) -> int {
      if (!v.empty()) KS_CUDA(cudaMemcpyAsync(buf.p, v.data(), v.size() * sizeof(v[0]), cudaMemcpyHostToDevice, u));
      return KS_OK;
    };
    if (int rc = put(f->rank_d, rk)) return rc;
    if (int rc = put(f->skel_pos, sp)) return rc;
    if (int rc = put(f->skel_off, so)) return rc;
    if (int rc = put(f->coeff_off, co)) return rc;
    if (int rc = put(f->leaf_node, ln)) return rc;
    if (int rc = put(f->leaf_begin, lbg)) return rc;
    if (int rc = put(f->leaf_size, lsz)) return rc;
    if (int rc = put(f->int_node, inode)) return rc;
    if (int rc = put(f->int_left, ileft)) return rc;
    if (int rc = put(f->int_right, iright)) return rc;
    double* orig = nullptr;
    int64_t* pmd = nullptr;
    KS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&orig), sizeof(double) * p->n * p->d, u));
    KS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&pmd), sizeof(int64_t) * p->n, u));
    KS_CUDA(cudaMemsetAsync(f->coords.p + (size_t)p->n * p->d, 0, sizeof(double) * f->m_pad * p->d, u));
    KS_CUDA(cudaMemcpyAsync(orig, p->coords, sizeof(double) * p->n * p->d, cudaMemcpyHostToDevice, u));
    KS_CUDA(cudaMemcpyAsync(pmd, p->perm, sizeof(int64_t) * p->n, cudaMemcpyHostToDevice, u));
    ks::launch_gather_rows(orig, pmd, p->n, p->d, f->coords.p, u);
    ks::launch_row_sqnorms(f->coords.p, p->n + f->m_pad, p->d, f->xx.p, u);
    KS_CUDA(cudaFreeAsync(orig, u));
    KS_CUDA(cudaFreeAsync(pmd, u));
    KS_CUDA(cudaEventRecord(f->ev_up_coords, u));
    // P blocks: leaves in leaf order (a milestone event per leaf quarter), then
    // internal nodes level by level, deepest first (an event per level), then
    // whatever this handle does not factor; contiguous ranges are coalesced
    std::vector<char> sent(nn, 0);
    int64_t r0 = -1, r1 = -1;
    auto flush = [&]() -> int {
      if (r1 > r0) KS_CUDA(cudaMemcpyAsync(f->coeff.p + r0, p->coeff + r0, sizeof(double) * (r1 - r0),
                                           cudaMemcpyHostToDevice, u));
      r0 = r1 = -1;
      return KS_OK;
    };
    auto add = [&](int64_t v) -> int {
      sent[v] = 1;
      const int64_t a0 = p->coeff_off[v], a1 = p->coeff_off[v + 1];
      if (a1 <= a0) return KS_OK;
      if (a0 == r1) { r1 = a1; return KS_OK; }
      if (int rc = flush()) return rc;
      r0 = a0;
      r1 = a1;
      return KS_OK;
    };
    for (int c = 0; c < ks_factor::kLeafChunks; ++c) {
      const size_t l0 = nl * c / ks_factor::kLeafChunks, l1 = nl * (c + 1) / ks_factor::kLeafChunks;
      for (size_t li = l0; li < l1; ++li)
        if (int rc = add(f->leaf_nodes[li])) return rc;
      if (int rc = flush()) return rc;
      KS_CUDA(cudaEventRecord(f->ev_up_leaf[c], u));
      // with subtree pipelining: then this subtree's nodes of the pipelined levels
      for (int lev = 0; lev < f->npipe; ++lev) {
        const auto& lv = f->levels[lev];
        const size_t c0 = lv.size() * c / ks_factor::kLeafChunks, c1 = lv.size() * (c + 1) / ks_factor::kLeafChunks;
        for (size_t i = c0; i < c1; ++i)
          if (int rc = add(lv[i])) return rc;
      }
      if (int rc = flush()) return rc;
      KS_CUDA(cudaEventRecord(f->ev_up_sub[c], u));
    }
    for (size_t lev = 0; lev < f->levels.size(); ++lev) {
      for (int v : f->levels[lev])
        if (!sent[v])
          if (int rc = add(v)) return rc;
      if (int rc = flush()) return rc;
      KS_CUDA(cudaEventRecord(f->ev_up_level[lev], u));
    }
    for (int64_t v = 0; v < nn; ++v)
      if (!sent[v])
        if (int rc = add(v)) return rc;
    if (int rc = flush()) return rc;
    KS_CUDA(cudaEventRecord(f->ev_up_all, u));
    f->upload_pending = true;
    return KS_OK;
  };
  if (int rc = start_uploads()) return abort_create(rc);
  const double t_issue = host_ms();
  // ---- host checks while the copies run: point coordinates on worker threads
  {
    const int64_t total = p->n * p->d;
    const int nth = (int)std::max<int64_t>(1, std::min<int64_t>(16, total / (1 << 20)));
    std::vector<char> ok(nth, 1);
    std::vector<std::thread> th;
    for (int t = 0; t < nth; ++t)
      th.emplace_back([&, t]() {
        const int64_t a = total * t / nth, b = total * (t + 1) / nth;
        for (int64_t i = a; i < b; ++i)
          if (!std::isfinite(p->coords[i])) { ok[t] = 0; return; }
      });
    for (auto& x : th) x.join();
    for (char c : ok)
      if (!c) return abort_create(fail(KS_ERR_INVALID, "coords contain non-finite values"));
  }
  if (host_timing())
    std::fprintf(stderr, "[ks_create] plan %.1f tables+alloc %.1f issue %.1f checks %.1f ms (uploads in flight)\n",
                 t_plan - t_start, t_alloc - t_plan, t_issue - t_alloc, host_ms() - t_issue);
  *out = f;
  return KS_OK;
}

int ks_create(const ks_problem* p, int device, ks_factor** out) { return create_impl(p, device, 0, out); }

int ks_create_shard(const ks_problem* p, int device, int64_t shard_root, ks_factor** out) {
  return create_impl(p, device, shard_root, out);
}

// Enqueue the whole factorization on `st` (no host synchronization inside, so
// the sequence can be captured into a CUDA graph). Leaf Cholesky failures are
// recorded on the device and handled by the caller afterwards.
// Leaves [l0, l1): left-looking Cholesky of the (m+s) x m trapezoids in 64-column
// panels (panel update GEMM, 64x64 POTRF + inverse, panel TRSM as GEMM with the
// inverse), then H = L21 L21^T (solver.py:123-135).
// Leaves [l0, l1): K(X_leaf, X_leaf) + lam I (lower triangle) and the P rows of
// the trapezoid [[A], [P]].
// wait_p: on the first factorization, the upload milestone of these leaves' P
// blocks (the Gaussian blocks need only the points, so they start before it)
static int enqueue_leaf_assemble(ks_factor* f, Launcher& L, int l0, int l1, cudaEvent_t wait_p = nullptr) {
  if (l1 <= l0) return KS_OK;
  const ks::DevTree dt = f->devtree();
  const ks::LeafBatch all = f->leafbatch();
  ks::LeafBatch lb = all;
  lb.count = l1 - l0;
  lb.node = all.node + l0;
  lb.begin = all.begin + l0;
  lb.size = all.size + l0;
  lb.A = all.A + (int64_t)l0 * all.a_stride;
  const int M = f->m_pad;
  if ((f->d & 1) == 0) {
    // a DMMA Gram GEMM with the Gaussian epilogue
    GemmArgs g = mk(M, M, (int)f->d, lb.count, Operand{f->coords.p, f->d, f->d, lb.begin},
                    Operand{f->coords.p, f->d, f->d, lb.begin}, OperandW{lb.A, M, lb.a_stride, nullptr}, 1.0, 0.0);
    g.ge = ks::GaussEpi{f->xx.p, lb.begin, lb.size, f->lam_dev.p, f->h};
    ++L.count[0];
    cudaError_t e = ks::gemm_gauss(g, L.st);
    if (e != cudaSuccess) return fail(KS_ERR_CUDA, "leaf gauss gemm: %s", cudaGetErrorString(e));
    if (wait_p) KS_CUDA(cudaStreamWaitEvent(L.st, wait_p, 0));
    ks::launch_leaf_copy_p(dt, lb, L.st);
  } else {
    if (wait_p) KS_CUDA(cudaStreamWaitEvent(L.st, wait_p, 0));
    ks::launch_leaf_assemble(dt, lb, f->lam_dev.p, L.st);
  }
  L.count[0] += 1;
  return L.check("leaf_assemble");
}

// KS_UNFUSED_LEAF_TRSM=1: separate update and TRSM GEMMs per leaf panel (A/B check)
static bool unfused_leaf_trsm() {
  const char* e = std::getenv("KS_UNFUSED_LEAF_TRSM");
  return e && e[0] == '1';
}

static int enqueue_leaf_chol(ks_factor* f, Launcher& L, int l0, int l1) {
  const ks::LeafBatch all = f->leafbatch();
  ks::LeafBatch lb = all;
  lb.count = l1 - l0;
  lb.node = all.node + l0;
  lb.begin = all.begin + l0;
  lb.size = all.size + l0;
  lb.A = all.A + (int64_t)l0 * all.a_stride;
  const int nl = lb.count;
  const int M = f->m_pad, S = f->s_pad, R = f->R;
  const int64_t AS = lb.a_stride;
  double* leafA = lb.A;
  double* inv = f->inv.p + (int64_t)l0 * M * 64;
  int* info = f->leaf_info.p + l0;
  cudaStream_t st = L.st;
  const bool fused = !unfused_leaf_trsm();
  for (int j0 = 0; j0 < M; j0 += 64) {
    const Operand Einv{inv + (int64_t)(j0 / 64) * 64 * 64, 64, (int64_t)M * 64, nullptr};
    if (j0 > 0) {  // left-looking update of the panel (all rows, or just its diagonal block)
      Operand A{leafA + (int64_t)j0 * M, M, AS, nullptr};
      Operand B{leafA + (int64_t)j0 * M, M, AS, nullptr};
      OperandW C{leafA + (int64_t)j0 * M + j0, M, AS, nullptr};
      if (fused) {
        ++L.count[0];
        cudaError_t e = ks::gemm_small_tile(mk(64, 64, j0, nl, A, B, C, -1.0, 1.0), st);
        if (e != cudaSuccess) return fail(KS_ERR_CUDA, "leaf diagonal update: %s", cudaGetErrorString(e));
        if (int rc = L.check("leaf_update_diag")) return rc;
      } else {
        int rc = L.gemm(mk(R - j0, 64, j0, nl, A, B, C, -1.0, 1.0), false, true, "leaf_update");
        if (rc) return rc;
      }
    }
    ks::launch_potrf64(lb, j0, inv, info, st);
    ++L.count[0];
    if (int rc = L.check("potrf64")) return rc;
    if (R - j0 - 64 > 0) {
      OperandW C{leafA + (int64_t)(j0 + 64) * M + j0, M, AS, nullptr};
      if (fused && j0 > 0) {
        // rows below the diagonal block: update and TRSM (x L_jj^-T) in one GEMM
        Operand A{leafA + (int64_t)(j0 + 64) * M, M, AS, nullptr};
        Operand B{leafA + (int64_t)j0 * M, M, AS, nullptr};
        GemmArgs g = mk(R - j0 - 64, 64, j0, nl, A, B, C, -1.0, 1.0);
        g.E = Einv;
        ++L.count[0];
        cudaError_t e = ks::gemm_update_trsm(g, st);
        if (e != cudaSuccess) return fail(KS_ERR_CUDA, "leaf update+trsm gemm: %s", cudaGetErrorString(e));
        if (int rc = L.check("leaf_update_trsm")) return rc;
      } else {
        Operand A{leafA + (int64_t)(j0 + 64) * M + j0, M, AS, nullptr};
        int rc = L.gemm(mk(R - j0 - 64, 64, 64, nl, A, Einv, C, 1.0, 0.0), false, true, "leaf_trsm");
        if (rc) return rc;
      }
    }
  }
  if (S > 0 && f->n_int > 0) {
    Operand A{leafA + (int64_t)M * M, M, AS, nullptr};
    OperandW C{f->hbuf.p, S, (int64_t)S * S, lb.node};
    // SYRK: lower-triangular tiles only, then mirrored (H exactly symmetric, so
    // the reference's 0.5 (H + H^T) is the identity on it)
    GemmArgs g = mk(S, S, M, nl, A, A, C, 1.0, 0.0);
    g.tri = 1;
    int rc = L.gemm(g, false, true, "leaf_syrk");
    if (rc) return rc;
    ks::launch_mirror_lower(f->hbuf.p, (int64_t)S * S, lb.node, nl, S, st);
    ++L.count[0];
    if (int rc = L.check("sym_h")) return rc;
  }
  KS_CUDA(cudaGetLastError());
  return KS_OK;
}

static int enqueue_levels(ks_factor* f, cudaStream_t st, Launcher& L, int lev0, int lev1, int deferred_before = 0);
static int enqueue_level_body(ks_factor* f, Launcher& L, const ks::NodeBatch& nb, bool is_root_level);
static ks::NodeBatch sub_batch(const ks::NodeBatch& nb, int off, int cnt, int T, int S, int TP);
// subtree pipelining (ks_factor::npipe) in this factorization: the default 4
// node groups, not under the per-level profiler or the tracer (their level
// boundaries would blur); KS_PIPE=0 disables it
static bool pipelined(const ks_factor* f, int G) {
  const char* e = std::getenv("KS_PIPE");
  if (e && e[0] == '0') return false;
  return f->npipe > 0 && G == ks_factor::kLeafChunks && !f->profiling && !trace_on();
}

// node groups per phase (KS_GROUPS, default 2; tracing forces 1 so per-launch
// events stay on one stream)
static int n_groups() {
  if (trace_on()) return 1;
  const char* e = std::getenv("KS_GROUPS");
  const int g = e ? std::atoi(e) : 8;
  return std::max(1, std::min(g, ks_factor::kGroups));
}

static int enqueue_factorization(ks_factor* f, cudaStream_t st) {
  Launcher L{f, st, &f->launches[0]};
  const ks::DevTree dt = f->devtree();
  const ks::LeafBatch lb = f->leafbatch();
  const int nl = lb.count;
  auto mark = [&](cudaEvent_t e) -> int {
    if (f->profiling) KS_CUDA(cudaEventRecord(e, st));
    return KS_OK;
  };
  f->cur_tag = -1;
  if (int rc = mark(f->ev_phase[0])) return rc;
  KS_CUDA(cudaMemsetAsync(f->leaf_info.p, 0, sizeof(int) * nl, st));
  if (f->n_int) KS_CUDA(cudaMemsetAsync(f->int_info.p, 0, sizeof(int) * f->n_int, st));
  if (f->lu_sync.p) KS_CUDA(cudaMemsetAsync(f->lu_sync.p + (int64_t)4 * f->n_int, 0, sizeof(unsigned), st));
  // ---- leaves: assemble [[K + lam I], [P]] and factor, leaves split into
  // independent groups on their own streams; on the first factorization each
  // group waits only for the uploads of its own P blocks
  if (f->upload_pending) KS_CUDA(cudaStreamWaitEvent(st, f->ev_up_coords, 0));
  if (int rc = L.check("start")) return rc;
  bool pipe = false;
  if (int rc = mark(f->ev_phase[1])) return rc;
  {
    const int G = (nl >= 2 * 64) ? n_groups() : 1;
    pipe = pipelined(f, G);
    if (G > 1) {
      KS_CUDA(cudaEventRecord(f->gfork, st));
      for (int g = 0; g < G; ++g) KS_CUDA(cudaStreamWaitEvent(f->gst[g], f->gfork, 0));
    }
    for (int g = 0; g < G; ++g) {
      const int l0 = (int)((int64_t)nl * g / G), l1 = (int)((int64_t)nl * (g + 1) / G);
      cudaStream_t gs = (G > 1) ? f->gst[g] : st;
      cudaEvent_t wait_p = nullptr;
      if (f->upload_pending && l1 > l0) {
        int c = 0;  // the upload chunk holding this group's last leaf
        while ((int64_t)nl * (c + 1) / ks_factor::kLeafChunks <= l1 - 1) ++c;
        wait_p = f->ev_up_leaf[c];
      }
      Launcher Lg{f, gs, &f->launches[0]};
      if (int rc = enqueue_leaf_assemble(f, Lg, l0, l1, wait_p)) return rc;
      if (int rc = enqueue_leaf_chol(f, Lg, l0, l1)) return rc;
      if (pipe) {  // this subtree's nodes of the deepest npipe levels, on the same stream
        if (f->upload_pending) KS_CUDA(cudaStreamWaitEvent(gs, f->ev_up_sub[g], 0));
        for (int lev = 0; lev < f->npipe; ++lev) {
          f->cur_tag = lev;
          const ks::NodeBatch nb = f->nodebatch(lev);
          const int c = nb.count / G;
          if (int rc = enqueue_level_body(f, Lg, sub_batch(nb, g * c, c, f->T, f->s_pad, f->t_pad), false)) return rc;
        }
        f->cur_tag = -1;
      }
    }
    if (G > 1)
      for (int g = 0; g < G; ++g) {
        KS_CUDA(cudaEventRecord(f->gjoin[g], f->gst[g]));
        KS_CUDA(cudaStreamWaitEvent(st, f->gjoin[g], 0));
      }
  }
  KS_CUDA(cudaGetLastError());
  if (int rc = mark(f->ev_phase[2])) return rc;
  if (int rc = mark(f->ev_phase[3])) return rc;
  // ---- the shard's internal levels, deepest first (the pipelined ones are
  // done; their condition estimates are still to be launched) ----
  if (int rc = enqueue_levels(f, st, L, pipe ? f->npipe : 0, f->n_local_levels, pipe ? f->npipe : 0)) return rc;
  if (int rc = mark(f->ev_phase[4])) return rc;
  return KS_OK;
}

// Levels with at most KS_SLAB_MAX (default 4) nodes run the persistent
// per-node LU (lu_slab.cu); KS_SLAB_MAX=0 keeps the launch sequence everywhere.
static bool use_slab(const ks_factor* f, const ks::NodeBatch& nb) {
  const char* e = std::getenv("KS_SLAB_MAX");
  const int mx = e ? std::atoi(e) : 4;
  return nb.count <= mx && f->lu_sync.p && ks::slab_width(nb) > 0;
}

// batches of at most KS_SPINE_MAX (default 16) nodes carry the P^T columns
// through the recursive LU (rlu ext)
static int spine_max() {
  const char* e = std::getenv("KS_SPINE_MAX");
  return e ? std::atoi(e) : 16;
}

// One level's node work on L's stream for the node sub-batch nb (coupling,
// augmented assembly, recursive LU, U12 / Schur, pivot composition, H out).
static int enqueue_level_body(ks_factor* f, Launcher& L, const ks::NodeBatch& nb, bool is_root_level) {
  const ks::DevTree dt = f->devtree();
  const int S = f->s_pad;
  const int TP = f->t_pad, T = f->T;
  const int64_t TT = (int64_t)T * T, SS = (int64_t)S * S;
  const int cnt = nb.count;
  cudaStream_t st = L.st;
    ks::launch_coupling(dt, nb, st);
    ks::launch_aug_init(dt, nb, st);
    L.count[0] += 3;
    int rc = L.check("coupling/aug_init");
    if (rc) return rc;
    // Z12 = B H_r, Z21 = B^T H_l   (W G, solver.py:142-148, zero blocks skipped)
    rc = L.gemm(mk(S, S, S, cnt, Operand{nb.Bc, S, SS, nullptr}, Operand{f->hbuf.p, S, SS, nb.right},
                   OperandW{nb.Aug + S, T, TT, nullptr}, 1.0, 0.0), false, true);
    if (rc) return rc;
    rc = L.gemm(mk(S, S, S, cnt, Operand{nb.Bc, S, SS, nullptr}, Operand{f->hbuf.p, S, SS, nb.left},
                   OperandW{nb.Aug + (int64_t)S * T, T, TT, nullptr}, 1.0, 0.0), true, true);
    if (rc) return rc;
    // -P G = [-P_l H_l, -P_r H_r]
    const int64_t PS = (int64_t)S * TP;
    rc = L.gemm(mk(S, S, S, cnt, Operand{nb.Pn, TP, PS, nullptr}, Operand{f->hbuf.p, S, SS, nb.left},
                   OperandW{nb.Aug + (int64_t)TP * T, T, TT, nullptr}, -1.0, 0.0), false, true);
    if (rc) return rc;
    rc = L.gemm(mk(S, S, S, cnt, Operand{nb.Pn + S, TP, PS, nullptr}, Operand{f->hbuf.p, S, SS, nb.right},
                   OperandW{nb.Aug + (int64_t)TP * T + S, T, TT, nullptr}, -1.0, 0.0), false, true);
    if (rc) return rc;
    if (use_slab(f, nb)) {
      // narrow level: the whole LU, U12, Schur block and H in one cooperative launch
      KS_CUDA(cudaMemsetAsync(nb.norm1, 0, sizeof(double) * cnt, st));
      unsigned* sy = f->lu_sync.p + (int64_t)4 * nb.first;
      KS_CUDA(cudaMemsetAsync(sy, 0, sizeof(unsigned) * 4 * cnt, st));
      if (ks::launch_lu_slab(nb, f->hbuf.p, SS, !is_root_level, sy, f->lu_sync.p + (int64_t)4 * f->n_int, st))
        return fail(KS_ERR_CUDA, "persistent LU launch failed: %s", cudaGetErrorString(cudaGetLastError()));
      ++L.count[0];
      if (int rc2 = L.check("lu_slab")) return rc2;
      ks::launch_compose_perm(nb, st);
      ++L.count[0];
      KS_CUDA(cudaGetLastError());
      return KS_OK;
    }
    ks::launch_colnorm1(dt, nb, st);
    ++L.count[0];
    if (int rc2 = L.check("colnorm1")) return rc2;
    // LU of the Z columns with pivots restricted to Z's rows
    int pend[4] = {0, 0, 0, 0};
    // ... with the P^T columns on the right spine of the recursion: U12 =
    // L^-1 Pi P^T and the Schur complement H = P G Z^-1 P^T come out of it
    // (small batches: fewer dependent launches; large batches keep the separate
    // U12 TRSM and Schur GEMM, which run at a higher tensor-pipe rate)
    const bool spine = nb.count <= spine_max();
    rc = rlu(L, nb, 0, TP, f->pw, pend, spine ? S : 0);
    if (rc) return rc;
    if (!spine) {
      rc = trsm_ul(L, nb, 0, TP, TP, S);
      if (rc) return rc;
      rc = L.gemm(mk(S, S, TP, cnt, Operand{nb.Aug + (int64_t)TP * T, T, TT, nullptr},
                     Operand{nb.Aug + TP, T, TT, nullptr}, OperandW{nb.Aug + (int64_t)TP * T + TP, T, TT, nullptr},
                     -1.0, 1.0), false, false);
      if (rc) return rc;
    }
    ks::launch_compose_perm(nb, st);
    ++L.count[0];
    if (!is_root_level) {
      ks::launch_extract_h(nb, f->hbuf.p, SS, st);
      ++L.count[0];
      if (int rc2 = L.check("extract_h")) return rc2;
    }
    KS_CUDA(cudaGetLastError());
  return KS_OK;
}

static ks::NodeBatch sub_batch(const ks::NodeBatch& nb, int off, int cnt, int T, int S, int TP) {
  ks::NodeBatch s = nb;
  s.count = cnt;
  s.first = nb.first + off;
  s.node = nb.node + off;
  s.left = nb.left + off;
  s.right = nb.right + off;
  s.Aug = nb.Aug + (int64_t)off * T * T;
  s.Bc = nb.Bc + (int64_t)off * S * S;
  s.Pn = nb.Pn + (int64_t)off * S * TP;
  s.piv = nb.piv + (int64_t)off * TP;
  s.norm1 = nb.norm1 + off;
  s.cond = nb.cond + off;
  s.info = nb.info + off;
  s.moves = nb.moves + (int64_t)off * (2 * 64 + 1);
  s.pm = nb.pm + (int64_t)off * TP;
  s.scratch = nb.scratch + (int64_t)off * 32 * 64;
  return s;
}

// SMs the overlapped condition estimates may occupy (of 148); KS_HAGER_CTAS overrides
static int hager_ctas() {
  const char* e = std::getenv("KS_HAGER_CTAS");
  return e ? std::max(1, std::atoi(e)) : 96;
}

// KS_HAGER_FLUSH=n: launch the deferred estimates at the first level with <= n
// nodes (default 0: the first narrow level, < 64 nodes)
static int hager_flush_nodes() {
  const char* e = std::getenv("KS_HAGER_FLUSH");
  return e ? std::atoi(e) : 0;
}

// KS_HAGER_SPLIT=0: narrow levels' estimates queue on `side` like the wide ones
static bool hager_split() {
  const char* e = std::getenv("KS_HAGER_SPLIT");
  return !(e && e[0] == '0');
}

// Internal levels [lev0, lev1) of the plan (deepest first); wide levels split
// into node groups on the group streams. Condition estimates run on the side
// stream (they only feed diagnostics), joined at the end. The estimates of the
// wide (HBM-heavy) levels wait for the first narrow level, whose latency-bound
// launches leave most SMs idle, instead of competing with the next wide level.
static int enqueue_levels(ks_factor* f, cudaStream_t st, Launcher& L, int lev0, int lev1, int deferred_before) {
  const ks::DevTree dt = f->devtree();
  auto mark = [&](cudaEvent_t e) -> int {
    if (f->profiling) KS_CUDA(cudaEventRecord(e, st));
    return KS_OK;
  };
  std::vector<int> deferred;  // levels whose estimate is not launched yet
  for (int lv = 0; lv < deferred_before; ++lv) deferred.push_back(lv);
  bool used_side = false, used_side2 = false;
  auto flush = [&]() -> int {
    if (deferred.empty()) return KS_OK;
    if (trace_on()) {  // inline, so the trace times each estimate
      for (int lv : deferred) {
        f->cur_tag = lv;
        ks::launch_hager(dt, f->nodebatch(lv), f->dinv.p, f->lut.p, 1 << 30, st);
        L.count[0] += ks::hager_launches(f->nodebatch(lv));
        if (int rc = L.check("hager")) return rc;
      }
      deferred.clear();
      return KS_OK;
    }
    KS_CUDA(cudaEventRecord(f->ev_fork, st));
    KS_CUDA(cudaStreamWaitEvent(f->side, f->ev_fork, 0));
    used_side = true;
    for (int lv : deferred) {
      ks::launch_hager(dt, f->nodebatch(lv), f->dinv.p, f->lut.p, hager_ctas(), f->side);
      L.count[0] += ks::hager_launches(f->nodebatch(lv));
    }
    deferred.clear();
    KS_CUDA(cudaGetLastError());
    return KS_OK;
  };
  for (int lev = lev0; lev < lev1; ++lev) {
    f->cur_tag = (int)lev;
    if (f->upload_pending) KS_CUDA(cudaStreamWaitEvent(st, f->ev_up_level[lev], 0));
    const ks::NodeBatch nb = f->nodebatch((int)lev);
    const bool is_root_level = (f->levels[lev][0] == 0);
    const bool wide = nb.count >= 64;
    if (hager_flush_nodes() > 0 ? nb.count <= hager_flush_nodes() : !wide)
      if (int rc = flush()) return rc;
    const int G = wide ? n_groups() : 1;
    if (G == 1) {
      if (int rc = enqueue_level_body(f, L, nb, is_root_level)) return rc;
    } else {
      KS_CUDA(cudaEventRecord(f->gfork, st));
      for (int g = 0; g < G; ++g) {
        KS_CUDA(cudaStreamWaitEvent(f->gst[g], f->gfork, 0));
        const int o0 = (int)((int64_t)nb.count * g / G), o1 = (int)((int64_t)nb.count * (g + 1) / G);
        Launcher Lg{f, f->gst[g], &f->launches[0]};
        if (int rc = enqueue_level_body(f, Lg, sub_batch(nb, o0, o1 - o0, f->T, f->s_pad, f->t_pad), is_root_level))
          return rc;
        KS_CUDA(cudaEventRecord(f->gjoin[g], f->gst[g]));
        KS_CUDA(cudaStreamWaitEvent(st, f->gjoin[g], 0));
      }
    }
    // condition estimate off the critical path: a narrow level's right away
    // on side2 (one CTA per node), a wide level's deferred (see above)
    if (!wide && !trace_on() && hager_split()) {
      KS_CUDA(cudaEventRecord(f->ev_fork2, st));
      KS_CUDA(cudaStreamWaitEvent(f->side2, f->ev_fork2, 0));
      used_side2 = true;
      ks::launch_hager(dt, nb, f->dinv.p, f->lut.p, nb.count, f->side2);
      L.count[0] += ks::hager_launches(nb);
      KS_CUDA(cudaGetLastError());
    } else {
      deferred.push_back(lev);
      if (hager_flush_nodes() > 0 ? nb.count <= hager_flush_nodes() : !wide)
        if (int rc = flush()) return rc;
    }
    if (int rc2 = mark(f->ev_level[lev])) return rc2;
  }
  if (int rc = flush()) return rc;
  if (used_side) {
    KS_CUDA(cudaEventRecord(f->ev_join, f->side));
    KS_CUDA(cudaStreamWaitEvent(st, f->ev_join, 0));
  }
  if (used_side2) {
    KS_CUDA(cudaEventRecord(f->ev_join2, f->side2));
    KS_CUDA(cudaStreamWaitEvent(st, f->ev_join2, 0));
  }
  return KS_OK;
}

// The reference raises at the first failing node in its processing order
// (levels bottom-up, ids ascending): singular LU (linalg.py:205-206), then the
// condition estimate above 1e14 (solver.py:150-152).
static int check_nodes(ks_factor* f, int k0, int k1) {
  for (int k = k0; k < k1; ++k) {
    if (f->int_info_h[k])
      return fail(KS_ERR_SINGULAR, "node %d: zero pivot column at elimination step %d", f->int_nodes[k],
                  f->int_info_h[k] - 1);
    const double cnd = f->cond_h[k];
    if (!(cnd <= kCondHard))
      return fail(KS_ERR_ILL_COND, "reduced system at node %d is numerically singular (1-norm condition estimate %.3e)",
                  f->int_nodes[k], cnd);
  }
  return KS_OK;
}

static bool force_leaf_lu() {
  const char* e = std::getenv("KS_FORCE_LEAF_LU");  // test hook: every leaf takes the LU path
  return e && e[0] == '1';
}

// Non-SPD leaves: LU with partial pivoting of [[A, -P^T], [P, 0]] for the
// first m_pad pivots (dense_factor(..., "lu-partial-pivot"), solver.py:127-130);
// the Schur complement is H = P A^-1 P^T (solver.py:134-135).
// device storage of the LU-fallback leaves listed in f->fb_leaf
static int fb_alloc(ks_factor* f) {
  const int nf = (int)f->fb_leaf.size();
  const int M = f->m_pad;
  const int T = M + ((f->n_nodes > 1) ? f->s_pad : 0);
  f->fb_aug.release(); f->fb_piv.release(); f->fb_info.release(); f->fb_moves.release(); f->fb_pm.release();
  f->fb_node.release(); f->fb_begin.release(); f->fb_size.release(); f->fb_norm1.release(); f->fb_cond.release();
  f->fb_y.release();
  f->fb_q = 0;
  f->fb_T = T;
  std::vector<int> nd, bg, sz;
  for (int li : f->fb_leaf) {
    const int v = f->leaf_nodes[li];
    nd.push_back(v);
    bg.push_back((int)f->begin[v]);
    sz.push_back((int)(f->end[v] - f->begin[v]));
  }
  KS_CUDA(f->fb_aug.alloc((size_t)nf * T * T));
  KS_CUDA(f->fb_piv.alloc((size_t)nf * M));
  KS_CUDA(f->fb_info.alloc(nf));
  KS_CUDA(f->fb_moves.alloc((size_t)nf * (2 * 64 + 1)));
  KS_CUDA(f->fb_pm.alloc((size_t)nf * M));
  KS_CUDA(f->fb_norm1.alloc(nf));
  KS_CUDA(f->fb_cond.alloc(nf));
  KS_CUDA(f->fb_node.upload(nd));
  KS_CUDA(f->fb_begin.upload(bg));
  KS_CUDA(f->fb_size.upload(sz));
  return KS_OK;
}

static int factor_fallback_leaves(ks_factor* f, cudaStream_t st) {
  const int nf = (int)f->fb_leaf.size();
  const int M = f->m_pad;
  const int S = (f->n_nodes > 1) ? f->s_pad : 0;
  const int T = M + S;
  if (nf == 0) return KS_OK;
  if (T != f->fb_T || f->fb_node.n != (size_t)nf)
    if (int rc = fb_alloc(f)) return rc;
  const ks::NodeBatch fb = f->fb_batch();
  Launcher L{f, st, &f->launches[0]};
  KS_CUDA(cudaMemsetAsync(f->fb_info.p, 0, sizeof(int) * nf, st));
  ks::launch_fb_assemble(f->devtree(), fb, f->fb_begin.p, f->fb_size.p, f->lam_dev.p, st);
  int pend[4] = {0, 0, 0, 0};
  int rc = rlu(L, fb, 0, M, T <= 1024 ? 16 : 8, pend, S);  // the -P^T columns on the spine: H comes out of it
  if (rc) return rc;
  if (S > 0) ks::launch_extract_h(fb, f->hbuf.p, (int64_t)f->s_pad * f->s_pad, st);
  ks::launch_compose_perm(fb, st);
  KS_CUDA(cudaGetLastError());
  std::vector<int> info(nf, 0);
  KS_CUDA(cudaMemcpyAsync(info.data(), f->fb_info.p, sizeof(int) * nf, cudaMemcpyDeviceToHost, st));
  KS_CUDA(cudaStreamSynchronize(st));
  for (int k = 0; k < nf; ++k)
    if (info[k])  // linalg.py:205-206 inside the fallback (solver.py:129)
      return fail(KS_ERR_SINGULAR, "leaf %d: zero pivot column at elimination step %d", f->leaf_nodes[f->fb_leaf[k]],
                  info[k] - 1);
  return KS_OK;
}

static int graph_mode() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("KS_GRAPH");
    v = e ? std::atoi(e) : 1;
  }
  return v;
}

int ks_factorize(ks_factor* f, double lam, void* stream) {
  if (!f) return fail(KS_ERR_INVALID, "null handle");
  if (!std::isfinite(lam) || lam < 0.0) return fail(KS_ERR_INVALID, "need lambda >= 0 and finite, got %g", lam);
  KS_CUDA(cudaSetDevice(f->device));
  cudaStream_t st = (cudaStream_t)stream;
  f->lam = lam;
  f->factored = false;
  f->launches[0] = 0;
  f->trace_n = 0;
  const int nl = (int)f->leaf_nodes.size();
  KS_CUDA(cudaMemcpyAsync(f->lam_dev.p, &f->lam, sizeof(double), cudaMemcpyHostToDevice, st));
  // CUDA graph of the ~1000-launch sequence: from the second factorization on
  // (KS_GRAPH=1, default), always (2) or never (0); tracing runs eagerly.
  const int gm = (trace_on() || debug_sync() || f->profiling) ? 0 : graph_mode();
  const bool use_graph = gm == 2 || (gm == 1 && f->n_factorizations > 0);
  if (use_graph && f->upload_pending) {  // a graph does not capture waits on the upload stream
    KS_CUDA(cudaStreamSynchronize(f->upl));
    f->upload_pending = false;
  }
  if (use_graph) {
    if (!f->graph_exec || f->graph_profiling != f->profiling) {
      if (f->graph_exec) { cudaGraphExecDestroy(f->graph_exec); f->graph_exec = nullptr; }
      cudaGraph_t g = nullptr;
      KS_CUDA(cudaStreamBeginCapture(f->cap, cudaStreamCaptureModeThreadLocal));
      int rc = enqueue_factorization(f, f->cap);
      cudaError_t ce = cudaStreamEndCapture(f->cap, &g);
      if (rc) { if (g) cudaGraphDestroy(g); return rc; }
      KS_CUDA(ce);
      KS_CUDA(cudaGraphInstantiate(&f->graph_exec, g, 0));
      cudaGraphDestroy(g);
      f->graph_profiling = f->profiling;
      f->graph_launches = f->launches[0];
    }
    KS_CUDA(cudaGraphLaunch(f->graph_exec, st));
    f->launches[0] = f->graph_launches;
  } else {
    int rc = enqueue_factorization(f, st);
    if (rc) return rc;
    if (f->upload_pending) {  // everything after this point sees every upload
      KS_CUDA(cudaStreamWaitEvent(st, f->ev_up_all, 0));
      f->upload_pending = false;
    }
  }
  ++f->n_factorizations;
  // leaf Cholesky failures (NotSPD) -> LU fallback for those leaves (solver.py:125-131)
  f->leaf_info_h.assign(nl, 0);
  KS_CUDA(cudaMemcpyAsync(f->leaf_info_h.data(), f->leaf_info.p, sizeof(int) * nl, cudaMemcpyDeviceToHost, st));
  KS_CUDA(cudaStreamSynchronize(st));
  f->fallback.clear();
  std::vector<int> failed;
  const bool force = force_leaf_lu();
  for (int i = 0; i < nl; ++i)
    if (f->leaf_info_h[i] || force) {
      f->fallback.push_back(f->leaf_nodes[i]);
      failed.push_back(i);
    }
  if (failed != f->fb_leaf) {
    f->fb_leaf = failed;
    f->fb_T = 0;  // re-plan the fallback buffers
  }
  if (!failed.empty()) {
    // LU for those leaves, then the internal levels again on the corrected H
    if (int rc = factor_fallback_leaves(f, st)) return rc;
    if (f->n_int) KS_CUDA(cudaMemsetAsync(f->int_info.p, 0, sizeof(int) * f->n_int, st));
    Launcher L{f, st, &f->launches[0]};
    if (int rc = enqueue_levels(f, st, L, 0, f->n_local_levels)) return rc;
  }
  // ---- diagnostics and errors (solver.py:150-152, 175-188) ----
  f->int_info_h.assign(f->n_int, 0);
  f->cond_h.assign(f->n_int, 0.0);
  if (f->n_int) {
    KS_CUDA(cudaMemcpyAsync(f->int_info_h.data(), f->int_info.p, sizeof(int) * f->n_int, cudaMemcpyDeviceToHost, st));
    KS_CUDA(cudaMemcpyAsync(f->cond_h.data(), f->cond.p, sizeof(double) * f->n_int, cudaMemcpyDeviceToHost, st));
  }
  unsigned watchdog = 0;
  if (f->lu_sync.p)
    KS_CUDA(cudaMemcpyAsync(&watchdog, f->lu_sync.p + (int64_t)4 * f->n_int, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  KS_CUDA(cudaStreamSynchronize(st));
  if (watchdog) return fail(KS_ERR_CUDA, "persistent LU: a node's slabs stopped making progress (watchdog)");
  if (f->profiling) {
    auto el = [](cudaEvent_t a, cudaEvent_t b) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, a, b);
      return (double)ms;
    };
    f->phase_ms[0] = el(f->ev_phase[0], f->ev_phase[1]);
    f->phase_ms[1] = el(f->ev_phase[1], f->ev_phase[2]);
    f->phase_ms[2] = el(f->ev_phase[2], f->ev_phase[3]);
    f->phase_ms[3] = el(f->ev_phase[3], f->ev_phase[4]);
    f->phase_ms[4] = el(f->ev_phase[0], f->ev_phase[4]);
    f->level_ms.assign(f->n_local_levels, 0.0);
    for (int i = 0; i < f->n_local_levels; ++i)
      f->level_ms[i] = el(i == 0 ? f->ev_phase[3] : f->ev_level[i - 1], f->ev_level[i]);
  }
  if (trace_on() && f->trace_n > 1) {
    std::vector<std::pair<std::string, std::pair<int, double>>> agg;
    for (int i = 1; i < f->trace_n; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, f->trace_ev[i - 1], f->trace_ev[i]);
      std::string nm = (f->trace_tag[i] < 0 ? std::string("leaf ") : "L" + std::to_string(f->trace_tag[i]) + " ") +
                       f->trace_name[i];
      bool found = false;
      for (auto& a : agg)
        if (a.first == nm) { a.second.first++; a.second.second += ms; found = true; }
      if (!found) agg.push_back({nm, {1, (double)ms}});
    }
    std::string rep;
    char line[160];
    for (auto& a : agg) {
      std::snprintf(line, sizeof line, "%-24s %5d x %10.3f ms\n", a.first.c_str(), a.second.first, a.second.second);
      rep += line;
    }
    rep += "-- last 120 launches --\n";
    for (int i = std::max(1, f->trace_n - 120); i < f->trace_n; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, f->trace_ev[i - 1], f->trace_ev[i]);
      std::snprintf(line, sizeof line, "%-18s %8.1f us\n", f->trace_name[i], ms * 1e3);
      rep += line;
    }
    f->trace_report = rep;
  }
  const int k1 = f->n_local_levels < (int)f->levels.size() ? f->level_first[f->n_local_levels] : f->n_int;
  if (int rc = check_nodes(f, 0, k1)) return rc;
  f->local_factored = true;
  f->factored = (f->n_local_levels == (int)f->levels.size());
  return KS_OK;
}

int ks_factorize_top(ks_factor* f, void* stream) {
  if (!f) return fail(KS_ERR_INVALID, "null handle");
  if (!f->local_factored) return fail(KS_ERR_INVALID, "factor the shard (ks_factorize) first");
  KS_CUDA(cudaSetDevice(f->device));
  cudaStream_t st = (cudaStream_t)stream;
  Launcher L{f, st, &f->launches[0]};
  if (int rc = enqueue_levels(f, st, L, f->n_local_levels, (int)f->levels.size())) return rc;
  const int k0 = f->n_local_levels < (int)f->levels.size() ? f->level_first[f->n_local_levels] : f->n_int;
  if (f->n_int > k0) {
    KS_CUDA(cudaMemcpyAsync(f->int_info_h.data() + k0, f->int_info.p + k0, sizeof(int) * (f->n_int - k0),
                            cudaMemcpyDeviceToHost, st));
    KS_CUDA(cudaMemcpyAsync(f->cond_h.data() + k0, f->cond.p + k0, sizeof(double) * (f->n_int - k0),
                            cudaMemcpyDeviceToHost, st));
  }
  KS_CUDA(cudaStreamSynchronize(st));
  if (int rc = check_nodes(f, k0, f->n_int)) return rc;
  f->factored = true;
  return KS_OK;
}

// ---- multi-RHS path (q >= kGemmSolveQ): factors applied as DMMA GEMMs ----
constexpr int64_t kGemmSolveQ = 8;

// op(T)^-1 B for an n x n triangle T (ld lda, batch stride sa) and B (n x ncols,
// ld ldb, batch stride sb): recursive halves, GEMM for the off-diagonal block,
// k_trsm_rhs at 8/16/32/64.
static int gemm_trsm(Launcher& L, bool upper, bool unit, const double* A, int64_t lda, int64_t sa, double* B,
                     int64_t ldb, int64_t sb, int n, int ncols, int batch) {
  if (n == 64 || n == 32 || n == 16 || n == 8) {
    ks::launch_trsm_rhs(n, upper, unit, A, lda, sa, B, ldb, sb, ncols, batch, L.st);
    ++*L.count;
    return L.check("trsm_rhs");
  }
  const int h = (n > 64) ? (int)roundup(n / 2, 8) : (n > 32 ? 32 : (n > 16 ? 16 : 8));
  int rc;
  if (!upper) {
    if ((rc = gemm_trsm(L, upper, unit, A, lda, sa, B, ldb, sb, h, ncols, batch))) return rc;
    rc = L.gemm(mk(n - h, ncols, h, batch, Operand{A + (int64_t)h * lda, lda, sa, nullptr}, Operand{B, ldb, sb, nullptr},
                   OperandW{B + (int64_t)h * ldb, ldb, sb, nullptr}, -1.0, 1.0), false, false);
    if (rc) return rc;
    return gemm_trsm(L, upper, unit, A + (int64_t)h * lda + h, lda, sa, B + (int64_t)h * ldb, ldb, sb, n - h, ncols,
                     batch);
  }
  if ((rc = gemm_trsm(L, upper, unit, A + (int64_t)h * lda + h, lda, sa, B + (int64_t)h * ldb, ldb, sb, n - h, ncols,
                      batch)))
    return rc;
  rc = L.gemm(mk(h, ncols, n - h, batch, Operand{A + h, lda, sa, nullptr}, Operand{B + (int64_t)h * ldb, ldb, sb, nullptr},
                 OperandW{B, ldb, sb, nullptr}, -1.0, 1.0), false, false);
  if (rc) return rc;
  return gemm_trsm(L, upper, unit, A, lda, sa, B, ldb, sb, h, ncols, batch);
}

// up pass at the leaves: z = L^-1 b (64-row blocks: GEMM update, then the block's
// stored inverse), c = L21 z
static int leaf_up_gemm(ks_factor* f, Launcher& L, const double* Bd, int q) {
  const ks::LeafBatch lb = f->leafbatch();
  const int nl = lb.count, M = f->m_pad, S = f->s_pad;
  const int64_t AS = lb.a_stride, ZS = (int64_t)M * q;
  ks::launch_leaf_gather(lb, Bd, q, f->z.p, q, L.st);
  ++*L.count;
  for (int r0 = 0; r0 < M; r0 += 64) {
    int rc;
    if (r0 > 0) {
      rc = L.gemm(mk(64, q, r0, nl, Operand{f->leafA.p + (int64_t)r0 * M, M, AS, nullptr}, Operand{f->z.p, q, ZS, nullptr},
                     OperandW{f->z.p + (int64_t)r0 * q, q, ZS, nullptr}, -1.0, 1.0), false, false);
      if (rc) return rc;
    }
    rc = L.gemm(mk(64, q, 64, nl, Operand{f->inv.p + (int64_t)(r0 / 64) * 4096, 64, (int64_t)M * 64, nullptr},
                   Operand{f->z.p + (int64_t)r0 * q, q, ZS, nullptr}, OperandW{f->z.p + (int64_t)r0 * q, q, ZS, nullptr},
                   1.0, 0.0), false, false);
    if (rc) return rc;
  }
  if (S > 0 && f->n_nodes > 1)
    return L.gemm(mk(S, q, M, nl, Operand{f->leafA.p + (int64_t)M * M, M, AS, nullptr}, Operand{f->z.p, q, ZS, nullptr},
                     OperandW{f->c.p, q, (int64_t)S * q, lb.node}, 1.0, 0.0), false, false);
  return KS_OK;
}

// down pass at the leaves: x = L^-T (z - L21^T t)
static int leaf_down_gemm(ks_factor* f, Launcher& L, double* Xd, int q) {
  const ks::LeafBatch lb = f->leafbatch();
  const int nl = lb.count, M = f->m_pad, S = f->s_pad;
  const int64_t AS = lb.a_stride, ZS = (int64_t)M * q;
  int rc;
  if (S > 0 && f->n_nodes > 1) {
    rc = L.gemm(mk(M, q, S, nl, Operand{f->leafA.p + (int64_t)M * M, M, AS, nullptr},
                   Operand{f->tin.p, q, (int64_t)S * q, lb.node}, OperandW{f->z.p, q, ZS, nullptr}, -1.0, 1.0),
                true, false);
    if (rc) return rc;
  }
  for (int r0 = M - 64; r0 >= 0; r0 -= 64) {
    if (r0 + 64 < M) {
      rc = L.gemm(mk(64, q, M - r0 - 64, nl, Operand{f->leafA.p + (int64_t)(r0 + 64) * M + r0, M, AS, nullptr},
                     Operand{f->z.p + (int64_t)(r0 + 64) * q, q, ZS, nullptr},
                     OperandW{f->z.p + (int64_t)r0 * q, q, ZS, nullptr}, -1.0, 1.0), true, false);
      if (rc) return rc;
    }
    rc = L.gemm(mk(64, q, 64, nl, Operand{f->inv.p + (int64_t)(r0 / 64) * 4096, 64, (int64_t)M * 64, nullptr},
                   Operand{f->z.p + (int64_t)r0 * q, q, ZS, nullptr}, OperandW{f->z.p + (int64_t)r0 * q, q, ZS, nullptr},
                   1.0, 0.0), true, false);
    if (rc) return rc;
  }
  ks::launch_leaf_scatter(lb, f->z.p, Xd, q, q, L.st);
  ++*L.count;
  return KS_OK;
}

// up pass at one level: w = [B c_r; B^T c_l], y = L^-1 Pi w, c = P cc + L21aug y
static int node_up_gemm(ks_factor* f, Launcher& L, const ks::NodeBatch& nb, bool root, int q) {
  const int S = f->s_pad, TP = f->t_pad, T = f->T, cnt = nb.count;
  const int64_t SS = (int64_t)S * S, TT = (int64_t)T * T, CS = (int64_t)S * q, YS = (int64_t)TP * q;
  double* w = f->wtmp.p + (int64_t)nb.first * YS;
  double* y = f->y.p + (int64_t)nb.first * YS;
  int rc = L.gemm(mk(S, q, S, cnt, Operand{nb.Bc, S, SS, nullptr}, Operand{f->c.p, q, CS, nb.right},
                     OperandW{w, q, YS, nullptr}, 1.0, 0.0), false, false);
  if (rc) return rc;
  rc = L.gemm(mk(S, q, S, cnt, Operand{nb.Bc, S, SS, nullptr}, Operand{f->c.p, q, CS, nb.left},
                 OperandW{w + (int64_t)S * q, q, YS, nullptr}, 1.0, 0.0), true, false);
  if (rc) return rc;
  ks::launch_permute_rows(nb, f->wtmp.p, f->y.p, q, L.st);
  ++*L.count;
  if ((rc = gemm_trsm(L, false, true, nb.Aug, T, TT, y, q, YS, TP, q, cnt))) return rc;
  if (root) return KS_OK;
  const int64_t PS = (int64_t)S * TP;
  rc = L.gemm(mk(S, q, S, cnt, Operand{nb.Pn, TP, PS, nullptr}, Operand{f->c.p, q, CS, nb.left},
                 OperandW{f->c.p, q, CS, nb.node}, 1.0, 0.0), false, false);
  if (rc) return rc;
  rc = L.gemm(mk(S, q, S, cnt, Operand{nb.Pn + S, TP, PS, nullptr}, Operand{f->c.p, q, CS, nb.right},
                 OperandW{f->c.p, q, CS, nb.node}, 1.0, 1.0), false, false);
  if (rc) return rc;
  return L.gemm(mk(S, q, TP, cnt, Operand{nb.Aug + (int64_t)TP * T, T, TT, nullptr}, Operand{y, q, YS, nullptr},
                   OperandW{f->c.p, q, CS, nb.node}, 1.0, 1.0), false, false);
}

// down pass at one level: u = U^-1 (y + U12aug t); children get split(u)
static int node_down_gemm(ks_factor* f, Launcher& L, const ks::NodeBatch& nb, bool root, int q) {
  const int S = f->s_pad, TP = f->t_pad, T = f->T, cnt = nb.count;
  const int64_t TT = (int64_t)T * T, CS = (int64_t)S * q, YS = (int64_t)TP * q;
  double* y = f->y.p + (int64_t)nb.first * YS;
  int rc;
  if (!root) {
    rc = L.gemm(mk(TP, q, S, cnt, Operand{nb.Aug + TP, T, TT, nullptr}, Operand{f->tin.p, q, CS, nb.node},
                   OperandW{y, q, YS, nullptr}, 1.0, 1.0), false, false);
    if (rc) return rc;
  }
  if ((rc = gemm_trsm(L, true, false, nb.Aug, T, TT, y, q, YS, TP, q, cnt))) return rc;
  ks::launch_split_u(nb, f->y.p, f->tin.p, q, L.st);
  ++*L.count;
  return KS_OK;
}

// LU-fallback leaves overwrite their Cholesky-path results (c at the leaf, x rows)
static int fb_up(ks_factor* f, const double* Bd, int64_t q, cudaStream_t st) {
  if (f->fb_leaf.empty()) return KS_OK;
  if (q > f->fb_q) {
    f->fb_y.release();
    KS_CUDA(f->fb_y.alloc((size_t)f->fb_leaf.size() * f->m_pad * q));
    f->fb_q = q;
  }
  ks::launch_fb_up(f->fb_batch(), f->fb_begin.p, f->fb_size.p, Bd, q, f->fb_y.p, f->c.p, (int)q, st);
  KS_CUDA(cudaGetLastError());
  return KS_OK;
}

static int fb_down(ks_factor* f, double* Xd, int64_t q, cudaStream_t st) {
  if (f->fb_leaf.empty()) return KS_OK;
  ks::launch_fb_down(f->fb_batch(), f->fb_begin.p, f->fb_size.p, f->fb_y.p, f->tin.p, Xd, q, (int)q, f->n_nodes > 1,
                     st);
  KS_CUDA(cudaGetLastError());
  return KS_OK;
}

static void trace_mark(ks_factor* f, cudaStream_t st, const char* what) {
  Launcher L{f, st, &f->launches[1]};
  L.check(what);
}

static void trace_build_report(ks_factor* f) {
  if (!trace_on() || f->trace_n < 2) return;
  cudaDeviceSynchronize();
  std::vector<std::pair<std::string, std::pair<int, double>>> agg;
  for (int i = 1; i < f->trace_n; ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, f->trace_ev[i - 1], f->trace_ev[i]);
    std::string nm = (f->trace_tag[i] < 0 ? std::string("leaf ") : "L" + std::to_string(f->trace_tag[i]) + " ") +
                     f->trace_name[i];
    bool found = false;
    for (auto& a : agg)
      if (a.first == nm) { a.second.first++; a.second.second += ms; found = true; }
    if (!found) agg.push_back({nm, {1, (double)ms}});
  }
  std::string rep;
  char line[160];
  for (auto& a : agg) {
    std::snprintf(line, sizeof line, "%-24s %5d x %10.3f ms\n", a.first.c_str(), a.second.first, a.second.second);
    rep += line;
  }
  f->trace_report = rep;
}

// Solve phases. Shard-local rows are [loc_begin, loc_end) of tree order; the
// kernels index B and X by absolute tree position, so local buffers are passed
// with a virtual base (ptr - loc_begin * q).
static int solve_up(ks_factor* f, const double* Bd, int64_t q, cudaStream_t st) {
  if (q >= kGemmSolveQ && (q & 1) == 0) {  // DMMA tiles need an even q
    Launcher L{f, st, &f->launches[1]};
    if (int rc = leaf_up_gemm(f, L, Bd, (int)q)) return rc;
    if (int rc = fb_up(f, Bd, q, st)) return rc;
    for (int lev = 0; lev < f->n_local_levels; ++lev)
      if (int rc = node_up_gemm(f, L, f->nodebatch(lev), f->levels[lev][0] == 0, (int)q)) return rc;
    KS_CUDA(cudaGetLastError());
    return KS_OK;
  }
  ks::SolveBufs sb{(int)q, f->z.p, f->c.p, f->tin.p, f->y.p};
  f->cur_tag = -1;
  trace_mark(f, st, "start");
  ks::launch_leaf_fwd(f->leafbatch(), Bd, q, sb, st);
  if (int rc = fb_up(f, Bd, q, st)) return rc;
  ++f->launches[1];
  trace_mark(f, st, "leaf_fwd");
  for (int lev = 0; lev < f->n_local_levels; ++lev) {
    f->cur_tag = lev;
    ks::launch_node_up(f->nodebatch(lev), sb, f->levels[lev][0] == 0, st);
    ++f->launches[1];
    trace_mark(f, st, "node_up");
  }
  KS_CUDA(cudaGetLastError());
  return KS_OK;
}

static int solve_top(ks_factor* f, int64_t q, cudaStream_t st) {
  if (q >= kGemmSolveQ && (q & 1) == 0) {  // DMMA tiles need an even q
    Launcher L{f, st, &f->launches[1]};
    const int nlev = (int)f->levels.size();
    for (int lev = f->n_local_levels; lev < nlev; ++lev)
      if (int rc = node_up_gemm(f, L, f->nodebatch(lev), f->levels[lev][0] == 0, (int)q)) return rc;
    for (int lev = nlev - 1; lev >= f->n_local_levels; --lev)
      if (int rc = node_down_gemm(f, L, f->nodebatch(lev), f->levels[lev][0] == 0, (int)q)) return rc;
    KS_CUDA(cudaGetLastError());
    return KS_OK;
  }
  ks::SolveBufs sb{(int)q, f->z.p, f->c.p, f->tin.p, f->y.p};
  const int nlev = (int)f->levels.size();
  for (int lev = f->n_local_levels; lev < nlev; ++lev) {
    ks::launch_node_up(f->nodebatch(lev), sb, f->levels[lev][0] == 0, st);
    ++f->launches[1];
  }
  for (int lev = nlev - 1; lev >= f->n_local_levels; --lev) {
    f->cur_tag = lev;
    ks::launch_node_down(f->nodebatch(lev), sb, f->levels[lev][0] == 0, st);
    ++f->launches[1];
    trace_mark(f, st, "node_down");
  }
  KS_CUDA(cudaGetLastError());
  return KS_OK;
}

static int solve_down(ks_factor* f, double* Xd, int64_t q, cudaStream_t st) {
  if (q >= kGemmSolveQ && (q & 1) == 0) {  // DMMA tiles need an even q
    Launcher L{f, st, &f->launches[1]};
    for (int lev = f->n_local_levels - 1; lev >= 0; --lev)
      if (int rc = node_down_gemm(f, L, f->nodebatch(lev), f->levels[lev][0] == 0, (int)q)) return rc;
    if (int rc = leaf_down_gemm(f, L, Xd, (int)q)) return rc;
    if (int rc = fb_down(f, Xd, q, st)) return rc;
    KS_CUDA(cudaGetLastError());
    return KS_OK;
  }
  ks::SolveBufs sb{(int)q, f->z.p, f->c.p, f->tin.p, f->y.p};
  for (int lev = f->n_local_levels - 1; lev >= 0; --lev) {
    f->cur_tag = lev;
    ks::launch_node_down(f->nodebatch(lev), sb, f->levels[lev][0] == 0, st);
    ++f->launches[1];
    trace_mark(f, st, "node_down");
  }
  f->cur_tag = -1;
  ks::launch_leaf_bwd(f->leafbatch(), Xd, q, sb, f->n_nodes > 1, st);
  if (int rc = fb_down(f, Xd, q, st)) return rc;
  ++f->launches[1];
  trace_mark(f, st, "leaf_bwd");
  KS_CUDA(cudaGetLastError());
  return KS_OK;
}

int ks_solve(ks_factor* f, const double* B, double* X, int64_t q, void* stream) {
  if (!f) return fail(KS_ERR_INVALID, "null handle");
  if (!f->factored) return fail(KS_ERR_INVALID, "handle is not factored");
  if (f->shard_root != 0) return fail(KS_ERR_INVALID, "sharded handle: use ks_solve_up / ks_solve_top / ks_solve_down");
  if (q < 0) return fail(KS_ERR_INVALID, "q must be >= 0");
  if (q == 0) return KS_OK;
  if (!B || !X) return fail(KS_ERR_INVALID, "null B or X");
  KS_CUDA(cudaSetDevice(f->device));
  cudaStream_t st = (cudaStream_t)stream;
  int rc = ensure_solve_bufs(f, q);
  if (rc) return rc;
  f->launches[1] = 0;
  f->trace_n = 0;
  PhaseTimer tm(f->profiling, st, 2);
  tm.mark(0);
  const bool bdev = is_device_ptr(B), xdev = is_device_ptr(X);
  const double* Bd = B;
  double* Xd = X;
  const size_t bytes = (size_t)f->n * q * sizeof(double);
  if (!bdev) {
    KS_CUDA(cudaMemcpyAsync(f->bdev.p, B, bytes, cudaMemcpyHostToDevice, st));
    Bd = f->bdev.p;
  }
  if (!xdev) Xd = f->xdev.p;
  if ((rc = solve_up(f, Bd, q, st))) return rc;
  if ((rc = solve_top(f, q, st))) return rc;
  if ((rc = solve_down(f, Xd, q, st))) return rc;
  if (!xdev) KS_CUDA(cudaMemcpyAsync(X, Xd, bytes, cudaMemcpyDeviceToHost, st));
  tm.mark(1);
  if (!xdev || !bdev) KS_CUDA(cudaStreamSynchronize(st));
  trace_build_report(f);
  if (f->profiling) {
    KS_CUDA(cudaStreamSynchronize(st));
    f->phase_ms[5] = tm.between(0, 1);
  }
  return KS_OK;
}

int ks_solve_up(ks_factor* f, const double* B_local, int64_t q, void* stream) {
  if (!f || !f->local_factored) return fail(KS_ERR_INVALID, "shard is not factored");
  if (q <= 0 || !B_local) return fail(KS_ERR_INVALID, "need q >= 1 and a device B");
  KS_CUDA(cudaSetDevice(f->device));
  if (int rc = ensure_solve_bufs(f, q)) return rc;
  f->launches[1] = 0;
  return solve_up(f, B_local - f->loc_begin * q, q, (cudaStream_t)stream);
}

int ks_solve_top(ks_factor* f, int64_t q, void* stream) {
  if (!f || !f->factored) return fail(KS_ERR_INVALID, "handle is not factored (ks_factorize_top)");
  KS_CUDA(cudaSetDevice(f->device));
  return solve_top(f, q, (cudaStream_t)stream);
}

int ks_solve_down(ks_factor* f, double* X_local, int64_t q, void* stream) {
  if (!f || !f->factored) return fail(KS_ERR_INVALID, "handle is not factored");
  if (q <= 0 || !X_local) return fail(KS_ERR_INVALID, "need q >= 1 and a device X");
  KS_CUDA(cudaSetDevice(f->device));
  return solve_down(f, X_local - f->loc_begin * q, q, (cudaStream_t)stream);
}

// Skeleton-sized exchange buffers of one node (device pointers): 0 = H
// (s_pad x s_pad), 1 = c (up-pass skeleton weights, s_pad x q), 2 = t (incoming
// down-pass vector, s_pad x q). dir 0 copies out of the handle, 1 into it.
int ks_node_exchange(ks_factor* f, int which, int64_t node, double* dev, int64_t q, int dir, void* stream) {
  if (!f || !dev || node < 0 || node >= f->n_nodes) return fail(KS_ERR_INVALID, "bad exchange arguments");
  KS_CUDA(cudaSetDevice(f->device));
  double* buf;
  size_t count;
  if (which == 0) {
    buf = f->hbuf.p + node * (int64_t)f->s_pad * f->s_pad;
    count = (size_t)f->s_pad * f->s_pad;
  } else {
    if (q > f->q_cap) return fail(KS_ERR_INVALID, "solve buffers hold q <= %lld", (long long)f->q_cap);
    buf = (which == 1 ? f->c.p : f->tin.p) + node * (int64_t)f->s_pad * q;
    count = (size_t)f->s_pad * q;
  }
  if (dir == 0)
    KS_CUDA(cudaMemcpyAsync(dev, buf, count * sizeof(double), cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  else
    KS_CUDA(cudaMemcpyAsync(buf, dev, count * sizeof(double), cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return KS_OK;
}

int ks_shard_info(const ks_factor* f, int64_t* out, int64_t cap) {
  // [shard_root, shard_level, loc_begin, loc_end, s_pad, n_peers, peers...]
  if (!f || !out) return fail(KS_ERR_INVALID, "null argument");
  std::vector<int64_t> v{f->shard_root, f->shard_level, f->loc_begin, f->loc_end, f->s_pad, (int64_t)f->peers.size()};
  for (int64_t p : f->peers) v.push_back(p);
  for (int64_t i = 0; i < (int64_t)v.size() && i < cap; ++i) out[i] = v[i];
  return (int)v.size();
}

// Y = K~ W, the compressed operator (hss_matvec, compress.py:352-411), on the
// handle's resident inputs and coupling blocks (needs a factorized handle).
int ks_matvec(ks_factor* f, const double* W, double* Y, int64_t q, void* stream) {
  if (!f || !f->factored) return fail(KS_ERR_INVALID, "handle is not factored");
  if (f->shard_root != 0) return fail(KS_ERR_INVALID, "matvec on a sharded handle is not supported");
  if (q < 0) return fail(KS_ERR_INVALID, "q must be >= 0");
  if (q == 0) return KS_OK;
  KS_CUDA(cudaSetDevice(f->device));
  cudaStream_t st = (cudaStream_t)stream;
  if (int rc = ensure_solve_bufs(f, q)) return rc;
  if (q > f->mv_q) {
    f->mv_c.release(); f->mv_inc.release(); f->mv_tot.release();
    const size_t cnt = (size_t)std::max<int64_t>(f->n_nodes * f->s_pad * q, 1);
    KS_CUDA(f->mv_c.alloc(cnt));
    KS_CUDA(f->mv_inc.alloc(cnt));
    KS_CUDA(f->mv_tot.alloc(cnt));
    f->mv_q = q;
  }
  const size_t vb = (size_t)f->n_nodes * f->s_pad * q * sizeof(double);
  KS_CUDA(cudaMemsetAsync(f->mv_c.p, 0, vb, st));
  KS_CUDA(cudaMemsetAsync(f->mv_inc.p, 0, vb, st));
  KS_CUDA(cudaMemsetAsync(f->mv_tot.p, 0, vb, st));
  const bool wdev = is_device_ptr(W), ydev = is_device_ptr(Y);
  const size_t bytes = (size_t)f->n * q * sizeof(double);
  const double* Wd = W;
  double* Yd = Y;
  if (!wdev) {
    KS_CUDA(cudaMemcpyAsync(f->bdev.p, W, bytes, cudaMemcpyHostToDevice, st));
    Wd = f->bdev.p;
  }
  if (!ydev) Yd = f->xdev.p;
  const ks::DevTree dt = f->devtree();
  const ks::LeafBatch lb = f->leafbatch();
  const int S = f->s_pad, nlev = (int)f->levels.size();
  if (S > 0) ks::launch_mv_up_leaf(dt, lb, Wd, q, f->mv_c.p, S, (int)q, st);
  for (int lev = 0; lev < nlev; ++lev) ks::launch_mv_up_node(dt, f->nodebatch(lev), f->mv_c.p, S, (int)q, st);
  for (int lev = 0; lev < nlev; ++lev) ks::launch_mv_couple(dt, f->nodebatch(lev), f->mv_c.p, f->mv_inc.p, S, (int)q, st);
  for (int lev = nlev - 1; lev >= 0; --lev)
    ks::launch_mv_down(dt, f->nodebatch(lev), f->mv_inc.p, f->mv_tot.p, S, (int)q, f->levels[lev][0] != 0, st);
  ks::launch_mv_leaf(dt, lb, Wd, q, f->mv_tot.p, Yd, S, (int)q, nlev > 0, st);
  KS_CUDA(cudaGetLastError());
  if (!ydev) KS_CUDA(cudaMemcpyAsync(Y, Yd, bytes, cudaMemcpyDeviceToHost, st));
  if (!ydev || !wdev) KS_CUDA(cudaStreamSynchronize(st));
  return KS_OK;
}

int ks_kernel_matvec(const double* x_test, int64_t n_test, const double* x_train, int64_t n_train, int64_t d,
                     double bandwidth, const double* w, double* out, int device, void* stream) {
  if (n_test < 0 || n_train < 0 || d < 1) return fail(KS_ERR_INVALID, "bad sizes");
  if (!(bandwidth > 0.0) || !std::isfinite(bandwidth))
    return fail(KS_ERR_INVALID, "gaussian kernel needs bandwidth > 0, got %g", bandwidth);
  if (n_test == 0) return KS_OK;
  if (!x_test || !out || (n_train > 0 && (!x_train || !w))) return fail(KS_ERR_INVALID, "null argument");
  KS_CUDA(cudaSetDevice(device));
  cudaStream_t st = (cudaStream_t)stream;
  const bool odev = is_device_ptr(out);
  if (n_train == 0) {
    if (odev) KS_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * n_test, st));
    else std::fill(out, out + n_test, 0.0);
    return KS_OK;
  }
  // coordinates padded to an even dimension (16-byte cp.async rows), norms, weights
  const int64_t dp = d + (d & 1);
  DBuf<double> xt, xr, xx, yy, wd, part, od;
  KS_CUDA(xt.alloc((size_t)n_test * dp));
  KS_CUDA(xr.alloc((size_t)n_train * dp));
  KS_CUDA(xx.alloc((size_t)n_test));
  KS_CUDA(yy.alloc((size_t)n_train));
  KS_CUDA(wd.alloc((size_t)n_train));
  if (dp != d) {
    KS_CUDA(cudaMemsetAsync(xt.p, 0, sizeof(double) * n_test * dp, st));
    KS_CUDA(cudaMemsetAsync(xr.p, 0, sizeof(double) * n_train * dp, st));
  }
  KS_CUDA(cudaMemcpy2DAsync(xt.p, sizeof(double) * dp, x_test, sizeof(double) * d, sizeof(double) * d, n_test,
                            cudaMemcpyDefault, st));
  KS_CUDA(cudaMemcpy2DAsync(xr.p, sizeof(double) * dp, x_train, sizeof(double) * d, sizeof(double) * d, n_train,
                            cudaMemcpyDefault, st));
  KS_CUDA(cudaMemcpyAsync(wd.p, w, sizeof(double) * n_train, cudaMemcpyDefault, st));
  ks::launch_row_sqnorms(xt.p, n_test, dp, xx.p, st);
  ks::launch_row_sqnorms(xr.p, n_train, dp, yy.p, st);
  double* outd = out;
  if (!odev) {
    KS_CUDA(od.alloc((size_t)n_test));
    outd = od.p;
  }
  // test rows in blocks so that the partial sums stay within ~256 MB
  const int64_t tiles = (n_train + 63) / 64;
  const int64_t rows_blk = std::max<int64_t>(64, std::min<int64_t>(n_test, (int64_t(1) << 25) / tiles / 64 * 64));
  KS_CUDA(part.alloc((size_t)tiles * std::min(rows_blk, n_test)));
  for (int64_t r0 = 0; r0 < n_test; r0 += rows_blk) {
    const int m = (int)std::min(rows_blk, n_test - r0);
    GemmArgs g = mk(m, (int)n_train, (int)dp, 1, Operand{xt.p + r0 * dp, dp, 0, nullptr},
                    Operand{xr.p, dp, 0, nullptr}, OperandW{nullptr, 0, 0, nullptr}, 1.0, 0.0);
    g.ke = ks::KrrEpi{xx.p + r0, yy.p, wd.p, part.p, 1.0 / (-2.0 * bandwidth * bandwidth)};
    int nt = 0;
    cudaError_t e = ks::gemm_krr(g, &nt, st);
    if (e != cudaSuccess) return fail(KS_ERR_CUDA, "kernel matvec gemm: %s", cudaGetErrorString(e));
    ks::launch_sum_partials(part.p, nt, m, outd + r0, st);
  }
  KS_CUDA(cudaGetLastError());
  if (!odev) KS_CUDA(cudaMemcpyAsync(out, outd, sizeof(double) * n_test, cudaMemcpyDeviceToHost, st));
  KS_CUDA(cudaStreamSynchronize(st));  // buffers are released on return
  return KS_OK;
}

int ks_get_lam(const ks_factor* f, double* lam) {
  if (!f || !lam) return fail(KS_ERR_INVALID, "null argument");
  if (!f->factored) return fail(KS_ERR_INVALID, "handle is not factored");
  *lam = f->lam;
  return KS_OK;
}

int ks_get_diag(const ks_factor* f, ks_diag* out) {
  if (!f || !out) return fail(KS_ERR_INVALID, "null argument");
  out->cholesky_fallbacks = (int64_t)f->fallback.size();
  out->n_z_cond = f->n_int;
  out->n_warnings = 0;
  out->error_node = -1;
  out->error_cond = 0.0;
  out->max_z_cond = 0.0;
  for (int k = 0; k < (int)f->cond_h.size(); ++k) {
    if (f->cond_h[k] > kCondWarn) ++out->n_warnings;
    out->max_z_cond = std::max(out->max_z_cond, f->cond_h[k]);
    if (out->error_node < 0 && (f->int_info_h[k] || !(f->cond_h[k] <= kCondHard))) {
      out->error_node = f->int_nodes[k];
      out->error_cond = f->cond_h[k];
    }
  }
  return KS_OK;
}

int64_t ks_get_z_cond(const ks_factor* f, int64_t* nodes, double* conds, int64_t cap) {
  if (!f) return 0;
  std::vector<std::pair<int, double>> v;
  for (int k = 0; k < (int)f->cond_h.size(); ++k) v.push_back({f->int_nodes[k], f->cond_h[k]});
  std::sort(v.begin(), v.end());
  int64_t i = 0;
  for (; i < (int64_t)v.size() && i < cap; ++i) {
    nodes[i] = v[i].first;
    conds[i] = v[i].second;
  }
  return (int64_t)v.size();
}

int64_t ks_get_fallback_nodes(const ks_factor* f, int64_t* nodes, int64_t cap) {
  if (!f) return 0;
  for (int64_t i = 0; i < (int64_t)f->fallback.size() && i < cap; ++i) nodes[i] = f->fallback[i];
  return (int64_t)f->fallback.size();
}

int ks_get_node_h(const ks_factor* f, int64_t node, double* out) {
  if (!f || !out || node <= 0 || node >= f->n_nodes) return fail(KS_ERR_INVALID, "bad node");
  const int r = (int)f->rank[node];
  KS_CUDA(cudaSetDevice(f->device));
  KS_CUDA(cudaDeviceSynchronize());
  KS_CUDA(cudaMemcpy2D(out, sizeof(double) * r, f->hbuf.p + (int64_t)node * f->s_pad * f->s_pad,
                       sizeof(double) * f->s_pad, sizeof(double) * r, r, cudaMemcpyDeviceToHost));
  return KS_OK;
}

int ks_get_leaf_factor(const ks_factor* f, int64_t node, double* out) {
  if (!f || !out) return fail(KS_ERR_INVALID, "null argument");
  auto it = std::find(f->leaf_nodes.begin(), f->leaf_nodes.end(), (int)node);
  if (it == f->leaf_nodes.end()) return fail(KS_ERR_INVALID, "node %lld is not a leaf", (long long)node);
  const int li = (int)(it - f->leaf_nodes.begin());
  const int m = (int)(f->end[node] - f->begin[node]);
  KS_CUDA(cudaSetDevice(f->device));
  KS_CUDA(cudaDeviceSynchronize());
  KS_CUDA(cudaMemcpy2D(out, sizeof(double) * m, f->leafA.p + (int64_t)li * f->R * f->m_pad, sizeof(double) * f->m_pad,
                       sizeof(double) * m, m, cudaMemcpyDeviceToHost));
  for (int i = 0; i < m; ++i)
    for (int j = i + 1; j < m; ++j) out[(int64_t)i * m + j] = 0.0;
  return KS_OK;
}

int ks_debug_copy(const ks_factor* f, int which, int64_t index, double* out, int64_t count) {
  if (!f || !out) return fail(KS_ERR_INVALID, "null argument");
  const double* base = nullptr;
  int64_t stride = 0;
  switch (which) {
    case 0: base = f->z.p; stride = (int64_t)f->m_pad * f->q_cap; break;      // per leaf index
    case 1: base = f->c.p; stride = (int64_t)f->s_pad * f->q_cap; break;      // per node
    case 2: base = f->tin.p; stride = (int64_t)f->s_pad * f->q_cap; break;    // per node
    case 3: base = f->y.p; stride = (int64_t)f->t_pad * f->q_cap; break;      // per internal index
    case 4: base = f->aug.p; stride = (int64_t)f->T * f->T; break;            // per internal index
    case 5: base = f->leafA.p; stride = (int64_t)f->R * f->m_pad; break;      // per leaf index
    default: return fail(KS_ERR_INVALID, "bad buffer id");
  }
  KS_CUDA(cudaSetDevice(f->device));
  KS_CUDA(cudaDeviceSynchronize());
  KS_CUDA(cudaMemcpy(out, base + index * stride, sizeof(double) * std::min(count, stride), cudaMemcpyDeviceToHost));
  return KS_OK;
}

// Raw device address of an internal buffer (same ids as ks_debug_copy), for probes.
int64_t ks_debug_ptr(const ks_factor* f, int which) {
  if (!f) return 0;
  switch (which) {
    case 0: return (int64_t)f->z.p;
    case 1: return (int64_t)f->c.p;
    case 2: return (int64_t)f->tin.p;
    case 3: return (int64_t)f->y.p;
    case 4: return (int64_t)f->aug.p;
    case 5: return (int64_t)f->leafA.p;
    case 6: return (int64_t)f->hbuf.p;
    case 7: return (int64_t)f->leaf_node.p;
    default: return 0;
  }
}

int ks_debug_layout(const ks_factor* f, int64_t* out8) {
  if (!f || !out8) return fail(KS_ERR_INVALID, "null argument");
  out8[0] = f->m_pad; out8[1] = f->s_pad; out8[2] = f->t_pad; out8[3] = f->T;
  out8[4] = f->R; out8[5] = f->q_cap; out8[6] = f->n_int; out8[7] = (int64_t)f->leaf_nodes.size();
  return KS_OK;
}

int64_t ks_device_bytes(const ks_factor* f) {
  if (!f) return 0;
  int64_t b = 0;
  b += f->coords.n * 8 + f->coeff.n * 8 + f->leafA.n * 8 + f->inv.n * 8 + f->hbuf.n * 8 + f->aug.n * 8;
  b += f->bc.n * 8 + f->pn.n * 8 + f->z.n * 8 + f->c.n * 8 + f->tin.n * 8 + f->y.n * 8;
  b += f->bdev.n * 8 + f->xdev.n * 8;
  return b;
}

int ks_set_profiling(ks_factor* f, int on) {
  if (!f) return fail(KS_ERR_INVALID, "null handle");
  f->profiling = on != 0;
  return KS_OK;
}

int ks_get_phase_ms(const ks_factor* f, double* ms, int cap) {
  if (!f) return 0;
  int n = std::min(cap, 6);
  for (int i = 0; i < n; ++i) ms[i] = f->phase_ms[i];
  return n;
}

int ks_get_level_ms(const ks_factor* f, double* ms, int cap) {
  if (!f) return 0;
  const int n = std::min<int>(cap, (int)f->level_ms.size());
  for (int i = 0; i < n; ++i) ms[i] = f->level_ms[i];
  return n;
}

// Test hook for the batched DMMA GEMM (tools/gemm_probe.py, tests): strided
// batches, C = alpha op(A) op(B) + beta C.
int ks_test_gemm(int M, int N, int K, int batch, int tri, const double* A, const double* B, double* C,
                 int64_t lda, int64_t sa, int64_t ldb, int64_t sb, int64_t ldc, int64_t sc, double alpha, double beta,
                 int ta, int tb, void* stream) {
  // tri >= 2 is a probe hook: C batches indexed through the int array at address (tri - 2)... not used
  ks::GemmArgs g = mk(M, N, K, batch, Operand{A, lda, sa, nullptr}, Operand{B, ldb, sb, nullptr},
                      OperandW{C, ldc, sc, nullptr}, alpha, beta);
  g.tri = tri;
  cudaError_t e = ks::gemm(g, ta != 0, tb != 0, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(KS_ERR_CUDA, "gemm: %s", cudaGetErrorString(e));
  return KS_OK;
}

int ks_test_gemm_cidx(int M, int N, int K, int batch, const double* A, const double* B, double* C, const int* cidx,
                      int64_t lda, int64_t sa, int64_t ldb, int64_t sb, int64_t ldc, int64_t sc, int ta, int tb,
                      void* stream) {
  ks::GemmArgs g = mk(M, N, K, batch, Operand{A, lda, sa, nullptr}, Operand{B, ldb, sb, nullptr},
                      OperandW{C, ldc, sc, cidx}, 1.0, 0.0);
  cudaError_t e = ks::gemm(g, ta != 0, tb != 0, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(KS_ERR_CUDA, "gemm: %s", cudaGetErrorString(e));
  return KS_OK;
}

int ks_trace_report(const ks_factor* f, char* buf, int64_t len) {
  if (!f || !buf || len <= 0) return 0;
  std::snprintf(buf, (size_t)len, "%s", f->trace_report.c_str());
  return (int)f->trace_report.size();
}

int64_t ks_last_launches(const ks_factor* f, int which) {
  if (!f || which < 0 || which > 1) return 0;
  return f->launches[which];
}

// ---------------------------------------------------------------------------
// Persistence: operator inputs and factors (container.h format)
// ---------------------------------------------------------------------------
}  // extern "C"

namespace {

uint64_t problem_fingerprint(const ks_problem* p) {
  ks::Fingerprint fp;
  const int64_t nn = p->n_nodes;
  const int64_t hdr[3] = {p->n, p->d, nn};
  fp.add(hdr, sizeof hdr);
  fp.add(&p->bandwidth, sizeof(double));
  fp.add(p->coords, sizeof(double) * p->n * p->d);
  fp.add(p->perm, sizeof(int64_t) * p->n);
  for (const int64_t* a : {p->node_begin, p->node_end, p->node_left, p->node_right, p->rank})
    fp.add(a, sizeof(int64_t) * nn);
  fp.add(p->skel_off, sizeof(int64_t) * (nn + 1));
  fp.add(p->skel, sizeof(int64_t) * p->skel_off[nn]);
  fp.add(p->coeff_off, sizeof(int64_t) * (nn + 1));
  fp.add(p->coeff, sizeof(double) * p->coeff_off[nn]);
  return fp.h;
}

bool problem_ok(const ks_problem* p) {
  return p && p->n > 0 && p->d > 0 && p->n_nodes > 0 && p->coords && p->perm && p->node_begin && p->node_end &&
         p->node_left && p->node_right && p->rank && p->skel_off && p->coeff_off &&
         (p->skel_off[p->n_nodes] == 0 || p->skel) && (p->coeff_off[p->n_nodes] == 0 || p->coeff);
}

struct ProblemStore {
  std::vector<double> coords, coeff;
  std::vector<int64_t> perm, nb, ne, nl, nr, rank, so, skel, co;
};

constexpr size_t kStage = size_t(64) << 20;  // pinned staging for device <-> file

template <typename T>
int save_dev(ks::KfWriter& w, const char* name, const DBuf<T>& b, void* stage) {
  const uint32_t dt = sizeof(T) == 4 ? ks::KF_I32 : (std::is_same<T, double>::value ? ks::KF_F64 : ks::KF_I64);
  w.begin(name, dt, b.n);
  const size_t bytes = b.n * sizeof(T);
  for (size_t off = 0; off < bytes; off += kStage) {
    const size_t c = std::min(kStage, bytes - off);
    KS_CUDA(cudaMemcpy(stage, reinterpret_cast<const char*>(b.p) + off, c, cudaMemcpyDeviceToHost));
    w.put(stage, c);
  }
  w.end(bytes);
  return w.ok ? KS_OK : fail(KS_ERR_IO, "write failed (%s)", name);
}

template <typename T>
int load_dev(ks::KfReader& r, const char* name, DBuf<T>& b, void* stage) {
  const uint32_t dt = sizeof(T) == 4 ? ks::KF_I32 : (std::is_same<T, double>::value ? ks::KF_F64 : ks::KF_I64);
  const ks::KfEntry* e = r.find(name, dt);
  if (!e) return fail(KS_ERR_IO, "factor file: missing entry %s", name);
  if (e->count != b.n) return fail(KS_ERR_IO, "factor file: entry %s has %llu elements, expected %llu", name,
                                   (unsigned long long)e->count, (unsigned long long)b.n);
  const size_t per = kStage / sizeof(T);
  for (size_t first = 0; first < b.n; first += per) {
    const size_t c = std::min(per, b.n - first);
    if (!r.read(*e, stage, first, c)) return fail(KS_ERR_IO, "factor file: truncated entry %s", name);
    KS_CUDA(cudaMemcpy(b.p + first, stage, c * sizeof(T), cudaMemcpyHostToDevice));
  }
  return KS_OK;
}

struct Pinned {
  void* p = nullptr;
  ~Pinned() {
    if (p) cudaFreeHost(p);
  }
};

}  // namespace

extern "C" {

int ks_save_problem(const ks_problem* p, const char* path) {
  if (!problem_ok(p) || !path) return fail(KS_ERR_INVALID, "null or empty problem/path");
  const int64_t nn = p->n_nodes;
  ks::KfWriter w;
  if (!w.open(path, 1)) return fail(KS_ERR_IO, "cannot write %s", path);
  const int64_t hdr[3] = {p->n, p->d, nn};
  const uint64_t fpv = problem_fingerprint(p);
  w.entry("header", ks::KF_I64, hdr, 3);
  w.entry("bandwidth", ks::KF_F64, &p->bandwidth, 1);
  w.entry("coords", ks::KF_F64, p->coords, (uint64_t)(p->n * p->d));
  w.entry("perm", ks::KF_I64, p->perm, (uint64_t)p->n);
  w.entry("node_begin", ks::KF_I64, p->node_begin, (uint64_t)nn);
  w.entry("node_end", ks::KF_I64, p->node_end, (uint64_t)nn);
  w.entry("node_left", ks::KF_I64, p->node_left, (uint64_t)nn);
  w.entry("node_right", ks::KF_I64, p->node_right, (uint64_t)nn);
  w.entry("rank", ks::KF_I64, p->rank, (uint64_t)nn);
  w.entry("skel_off", ks::KF_I64, p->skel_off, (uint64_t)(nn + 1));
  w.entry("skel", ks::KF_I64, p->skel, (uint64_t)p->skel_off[nn]);
  w.entry("coeff_off", ks::KF_I64, p->coeff_off, (uint64_t)(nn + 1));
  w.entry("coeff", ks::KF_F64, p->coeff, (uint64_t)p->coeff_off[nn]);
  w.entry("fingerprint", ks::KF_I64, &fpv, 1);
  if (!w.close()) return fail(KS_ERR_IO, "write failed: %s", path);
  return KS_OK;
}

int ks_load_problem(const char* path, ks_problem* out, void** owner) {
  if (!path || !out || !owner) return fail(KS_ERR_INVALID, "null argument");
  *owner = nullptr;
  ks::KfReader r;
  if (!r.open(path)) return fail(KS_ERR_IO, "%s: %s", path, r.err.c_str());
  if (r.kind != 1) return fail(KS_ERR_IO, "%s: not an operator file", path);
  std::vector<int64_t> hdr;
  if (!r.read_vec("header", ks::KF_I64, hdr) || hdr.size() != 3 || hdr[0] < 1 || hdr[1] < 1 || hdr[2] < 1)
    return fail(KS_ERR_IO, "%s: bad header", path);
  const int64_t n = hdr[0], d = hdr[1], nn = hdr[2];
  auto* st = new ProblemStore();
  std::vector<double> bw;
  bool ok = r.read_vec("bandwidth", ks::KF_F64, bw) && bw.size() == 1 &&
            r.read_vec("coords", ks::KF_F64, st->coords) && (int64_t)st->coords.size() == n * d &&
            r.read_vec("perm", ks::KF_I64, st->perm) && (int64_t)st->perm.size() == n &&
            r.read_vec("node_begin", ks::KF_I64, st->nb) && (int64_t)st->nb.size() == nn &&
            r.read_vec("node_end", ks::KF_I64, st->ne) && (int64_t)st->ne.size() == nn &&
            r.read_vec("node_left", ks::KF_I64, st->nl) && (int64_t)st->nl.size() == nn &&
            r.read_vec("node_right", ks::KF_I64, st->nr) && (int64_t)st->nr.size() == nn &&
            r.read_vec("rank", ks::KF_I64, st->rank) && (int64_t)st->rank.size() == nn &&
            r.read_vec("skel_off", ks::KF_I64, st->so) && (int64_t)st->so.size() == nn + 1 &&
            r.read_vec("skel", ks::KF_I64, st->skel) && (int64_t)st->skel.size() == st->so[nn] &&
            r.read_vec("coeff_off", ks::KF_I64, st->co) && (int64_t)st->co.size() == nn + 1 &&
            r.read_vec("coeff", ks::KF_F64, st->coeff) && (int64_t)st->coeff.size() == st->co[nn];
  if (!ok) {
    delete st;
    return fail(KS_ERR_IO, "%s: missing or inconsistent operator entries", path);
  }
  ks_problem p{};
  p.n = n; p.d = d; p.n_nodes = nn;
  p.coords = st->coords.data(); p.perm = st->perm.data();
  p.node_begin = st->nb.data(); p.node_end = st->ne.data(); p.node_left = st->nl.data(); p.node_right = st->nr.data();
  p.rank = st->rank.data(); p.skel_off = st->so.data(); p.skel = st->skel.data();
  p.coeff_off = st->co.data(); p.coeff = st->coeff.data(); p.bandwidth = bw[0];
  std::vector<int64_t> fpv;
  if (r.read_vec("fingerprint", ks::KF_I64, fpv) && fpv.size() == 1 && (uint64_t)fpv[0] != problem_fingerprint(&p)) {
    delete st;
    return fail(KS_ERR_IO, "%s: fingerprint mismatch (corrupt file)", path);
  }
  *out = p;
  *owner = st;
  return KS_OK;
}

int ks_free_problem(void* owner) {
  delete static_cast<ProblemStore*>(owner);
  return KS_OK;
}

int ks_save_factor(const ks_factor* f, const ks_problem* p, const char* path) {
  if (!f || !path || !problem_ok(p)) return fail(KS_ERR_INVALID, "null argument");
  if (!f->factored) return fail(KS_ERR_INVALID, "handle is not factored");
  if (f->shard_root != 0) return fail(KS_ERR_UNSUPPORTED, "saving a sharded handle is not supported");
  if (p->n != f->n || p->d != f->d || p->n_nodes != f->n_nodes)
    return fail(KS_ERR_INVALID, "problem does not match the handle");
  KS_CUDA(cudaSetDevice(f->device));
  KS_CUDA(cudaDeviceSynchronize());
  Pinned stage;
  KS_CUDA(cudaMallocHost(&stage.p, kStage));
  ks::KfWriter w;
  if (!w.open(path, 2)) return fail(KS_ERR_IO, "cannot write %s", path);
  const uint64_t fpv = problem_fingerprint(p);
  const int64_t dims[9] = {f->m_pad, f->s_pad, f->t_pad, f->T, f->R, f->n_int, (int64_t)f->leaf_nodes.size(),
                           f->fb_T, (int64_t)f->fb_leaf.size()};
  w.entry("fingerprint", ks::KF_I64, &fpv, 1);
  w.entry("lam", ks::KF_F64, &f->lam, 1);
  w.entry("dims", ks::KF_I64, dims, 9);
  w.entry("leaf_info_h", ks::KF_I32, f->leaf_info_h.data(), f->leaf_info_h.size());
  w.entry("int_info_h", ks::KF_I32, f->int_info_h.data(), f->int_info_h.size());
  w.entry("cond_h", ks::KF_F64, f->cond_h.data(), f->cond_h.size());
  w.entry("fallback", ks::KF_I64, f->fallback.data(), f->fallback.size());
  w.entry("fb_leaf", ks::KF_I32, f->fb_leaf.data(), f->fb_leaf.size());
  void* sp = stage.p;
  int rc = save_dev(w, "leafA", f->leafA, sp);
  if (!rc) rc = save_dev(w, "inv", f->inv, sp);
  if (!rc) rc = save_dev(w, "hbuf", f->hbuf, sp);
  if (!rc) rc = save_dev(w, "aug", f->aug, sp);
  if (!rc) rc = save_dev(w, "bc", f->bc, sp);
  if (!rc) rc = save_dev(w, "pn", f->pn, sp);
  if (!rc) rc = save_dev(w, "piv", f->piv, sp);
  if (!rc) rc = save_dev(w, "pm", f->pm, sp);
  if (!rc) rc = save_dev(w, "norm1", f->norm1, sp);
  if (!rc) rc = save_dev(w, "cond", f->cond, sp);
  if (!rc) rc = save_dev(w, "leaf_info", f->leaf_info, sp);
  if (!rc) rc = save_dev(w, "int_info", f->int_info, sp);
  if (!rc && !f->fb_leaf.empty()) {
    rc = save_dev(w, "fb_aug", f->fb_aug, sp);
    if (!rc) rc = save_dev(w, "fb_piv", f->fb_piv, sp);
    if (!rc) rc = save_dev(w, "fb_pm", f->fb_pm, sp);
    if (!rc) rc = save_dev(w, "fb_info", f->fb_info, sp);
    if (!rc) rc = save_dev(w, "fb_norm1", f->fb_norm1, sp);
    if (!rc) rc = save_dev(w, "fb_cond", f->fb_cond, sp);
  }
  const bool closed = w.close();
  if (rc) return rc;
  if (!closed) return fail(KS_ERR_IO, "write failed: %s", path);
  return KS_OK;
}

int ks_load_factor(const char* path, const ks_problem* p, int device, ks_factor** out) {
  if (!path || !out || !problem_ok(p)) return fail(KS_ERR_INVALID, "null argument");
  *out = nullptr;
  ks::KfReader r;
  if (!r.open(path)) return fail(KS_ERR_IO, "%s: %s", path, r.err.c_str());
  if (r.kind != 2) return fail(KS_ERR_IO, "%s: not a factor file", path);
  std::vector<int64_t> fpv, dims;
  std::vector<double> lam;
  if (!r.read_vec("fingerprint", ks::KF_I64, fpv) || fpv.size() != 1 || !r.read_vec("dims", ks::KF_I64, dims) ||
      dims.size() != 9 || !r.read_vec("lam", ks::KF_F64, lam) || lam.size() != 1)
    return fail(KS_ERR_IO, "%s: bad factor header", path);
  if ((uint64_t)fpv[0] != problem_fingerprint(p))
    return fail(KS_ERR_INVALID, "%s: the factor was computed for a different operator", path);
  ks_factor* f = nullptr;
  if (int rc = create_impl(p, device, 0, &f)) return rc;
  if (cudaStreamSynchronize(f->upl) != cudaSuccess) {  // no factorization will wait for the uploads
    ks_destroy(f);
    return fail(KS_ERR_CUDA, "upload failed");
  }
  f->upload_pending = false;
  auto bad = [&](int rc) {
    ks_destroy(f);
    return rc;
  };
  const int64_t want[7] = {f->m_pad, f->s_pad, f->t_pad, f->T, f->R, f->n_int, (int64_t)f->leaf_nodes.size()};
  for (int i = 0; i < 7; ++i)
    if (dims[i] != want[i]) return bad(fail(KS_ERR_IO, "%s: factor layout differs from this library build", path));
  std::vector<int> fbl;
  if (!r.read_vec("leaf_info_h", ks::KF_I32, f->leaf_info_h) || !r.read_vec("int_info_h", ks::KF_I32, f->int_info_h) ||
      !r.read_vec("cond_h", ks::KF_F64, f->cond_h) || !r.read_vec("fallback", ks::KF_I64, f->fallback) ||
      !r.read_vec("fb_leaf", ks::KF_I32, fbl))
    return bad(fail(KS_ERR_IO, "%s: missing diagnostics", path));
  Pinned stage;
  KS_CUDA(cudaMallocHost(&stage.p, kStage));
  void* sp = stage.p;
  int rc = load_dev(r, "leafA", f->leafA, sp);
  if (!rc) rc = load_dev(r, "inv", f->inv, sp);
  if (!rc) rc = load_dev(r, "hbuf", f->hbuf, sp);
  if (!rc) rc = load_dev(r, "aug", f->aug, sp);
  if (!rc) rc = load_dev(r, "bc", f->bc, sp);
  if (!rc) rc = load_dev(r, "pn", f->pn, sp);
  if (!rc) rc = load_dev(r, "piv", f->piv, sp);
  if (!rc) rc = load_dev(r, "pm", f->pm, sp);
  if (!rc) rc = load_dev(r, "norm1", f->norm1, sp);
  if (!rc) rc = load_dev(r, "cond", f->cond, sp);
  if (!rc) rc = load_dev(r, "leaf_info", f->leaf_info, sp);
  if (!rc) rc = load_dev(r, "int_info", f->int_info, sp);
  if (!rc && !fbl.empty()) {
    f->fb_leaf = fbl;
    rc = fb_alloc(f);
    if (!rc) rc = load_dev(r, "fb_aug", f->fb_aug, sp);
    if (!rc) rc = load_dev(r, "fb_piv", f->fb_piv, sp);
    if (!rc) rc = load_dev(r, "fb_pm", f->fb_pm, sp);
    if (!rc) rc = load_dev(r, "fb_info", f->fb_info, sp);
    if (!rc) rc = load_dev(r, "fb_norm1", f->fb_norm1, sp);
    if (!rc) rc = load_dev(r, "fb_cond", f->fb_cond, sp);
  }
  if (rc) return bad(rc);
  f->lam = lam[0];
  if (cudaMemcpy(f->lam_dev.p, &f->lam, sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess)
    return bad(fail(KS_ERR_CUDA, "lam upload failed"));
  f->factored = true;
  f->local_factored = true;
  *out = f;
  return KS_OK;
}

void ks_destroy(ks_factor* f) {
  if (!f) return;
  cudaSetDevice(f->device);
  cudaDeviceSynchronize();
  f->release_all();
  if (f->graph_exec) cudaGraphExecDestroy(f->graph_exec);
  if (f->side) cudaStreamDestroy(f->side);
  if (f->side2) cudaStreamDestroy(f->side2);
  if (f->ev_fork2) cudaEventDestroy(f->ev_fork2);
  if (f->ev_join2) cudaEventDestroy(f->ev_join2);
  if (f->cap) cudaStreamDestroy(f->cap);
  for (auto g : f->gst)
    if (g) cudaStreamDestroy(g);
  if (f->gfork) cudaEventDestroy(f->gfork);
  for (auto e : f->gjoin)
    if (e) cudaEventDestroy(e);
  for (auto e : f->ev_phase)
    if (e) cudaEventDestroy(e);
  for (auto e : f->ev_level) cudaEventDestroy(e);
  for (auto e : f->trace_ev) cudaEventDestroy(e);
  f->lam_dev.release();
  if (f->ev_fork) cudaEventDestroy(f->ev_fork);
  if (f->ev_join) cudaEventDestroy(f->ev_join);
  if (f->upl) cudaStreamDestroy(f->upl);
  if (f->ev_up_coords) cudaEventDestroy(f->ev_up_coords);
  if (f->ev_up_all) cudaEventDestroy(f->ev_up_all);
  for (auto e : f->ev_up_leaf)
    if (e) cudaEventDestroy(e);
  for (auto e : f->ev_up_sub)
    if (e) cudaEventDestroy(e);
  for (auto e : f->ev_up_level)
    if (e) cudaEventDestroy(e);
  delete f;
}

}  // extern "C"
