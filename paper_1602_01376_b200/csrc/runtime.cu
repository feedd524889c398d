// Host runtime basics: error reporting, the device memory pool, tuning
// switches, the launch helper and the recursive LU / TRSM launch sequences
// shared by the factorization schedule (factorize.cu), and ks_destroy.
#include <ctime>

#include "handle.h"

namespace ksr {

namespace {
thread_local std::string g_err;
}

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

const std::string& last_error_msg() { return g_err; }

namespace {
int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return (e && e[0]) ? std::atoi(e) : dflt;
}
bool env_flag(const char* name, bool dflt) {
  const char* e = std::getenv(name);
  if (!e || !e[0]) return dflt;
  return e[0] == '1';
}
bool env_once(const char* name) {
  const char* e = std::getenv(name);
  return e && e[0] == '1';
}
}  // namespace

Knobs read_knobs() {
  Knobs k;
  k.slab_max = env_int("KS_SLAB_MAX", k.slab_max);
  k.spine_max = env_int("KS_SPINE_MAX", k.spine_max);
  k.groups = std::max(1, std::min(env_int("KS_GROUPS", k.groups), ks_factor::kGroups));
  k.pipe = env_flag("KS_PIPE", k.pipe);
  k.pipe_min = std::max(1, env_int("KS_PIPE_MIN", k.pipe_min));
  k.panel_w = env_int("KS_PANEL_W", 0);
  k.fused_merge = env_flag("KS_FUSED_MERGE", false);
  k.unfused_leaf_trsm = env_flag("KS_UNFUSED_LEAF_TRSM", false);
  k.split_leaf = env_flag("KS_SPLIT_LEAF", k.split_leaf);
  k.hager_ctas = std::max(1, env_int("KS_HAGER_CTAS", k.hager_ctas));
  k.hager_flush = env_int("KS_HAGER_FLUSH", k.hager_flush);
  k.hager_split = env_flag("KS_HAGER_SPLIT", k.hager_split);
  k.hager_early = env_flag("KS_HAGER_EARLY", k.hager_early);
  k.force_leaf_lu = env_flag("KS_FORCE_LEAF_LU", false);
  k.graph = env_int("KS_GRAPH", k.graph);
  k.ablate = env_int("KS_ABLATE", 0);
  return k;
}

bool trace_on() {
  static const bool v = env_once("KS_TRACE");
  return v;
}
bool debug_sync() {
  static const bool v = env_once("KS_DEBUG_SYNC");
  return v;
}
bool host_timing() {
  static const bool v = env_once("KS_HOST_TIMING");
  return v;
}

double host_ms() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

// ---- device memory ----
// Handle buffers come from a PRIVATE stream-ordered pool per device (not the
// device's default pool, which other libraries share). Like torch's caching
// allocator it keeps freed memory for the next handle by default (a new
// factorize call on the same shapes then maps no new memory: at config 5,
// ~80 GB of fresh mappings cost ~1 s); KS_POOL_GB caps what it keeps
// (fractional values allowed; 0 returns everything on every ks_destroy), and
// ks_trim_pool() (Python: release_cached_memory()) returns the cache to the
// driver. Frees keep the device-wide synchronization cudaFree implies
// (buffers may be in use on any stream).
namespace {
constexpr int kMaxDev = 64;
std::mutex g_pool_mu;
cudaMemPool_t g_pool[kMaxDev] = {};

double pool_keep_gb() {
  const char* env = std::getenv("KS_POOL_GB");
  if (!env || !env[0]) return -1.0;  // keep everything
  const double gb = std::atof(env);
  return gb > 0.0 ? gb : 0.0;
}

cudaError_t pool_get(cudaMemPool_t* out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDev) return cudaErrorInvalidDevice;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (!g_pool[dev]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool;
    if ((e = cudaMemPoolCreate(&pool, &props)) != cudaSuccess) return e;
    const double gb = pool_keep_gb();
    uint64_t keep = gb < 0.0 ? UINT64_MAX : (uint64_t)(gb * (double)(1ull << 30));
    if ((e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep)) != cudaSuccess) return e;
    g_pool[dev] = pool;
  }
  *out = g_pool[dev];
  return cudaSuccess;
}
}  // namespace

cudaError_t pool_alloc_async(void** p, size_t bytes, cudaStream_t st) {
  cudaMemPool_t pool;
  cudaError_t e = pool_get(&pool);
  if (e != cudaSuccess) return e;
  return cudaMallocFromPoolAsync(p, bytes, pool, st);
}

cudaError_t pool_alloc(void** p, size_t bytes) {
  cudaMemPool_t pool;
  cudaError_t e = pool_get(&pool);
  if (e != cudaSuccess) return e;
  if ((e = cudaMallocFromPoolAsync(p, bytes, pool, 0)) != cudaSuccess) return e;
  return cudaStreamSynchronize(0);  // usable from every stream once this returns
}

void pool_free(void* p) {
  cudaDeviceSynchronize();
  cudaFreeAsync(p, 0);
  cudaStreamSynchronize(0);
}

void pool_trim() {
  cudaMemPool_t pool;
  if (pool_get(&pool) != cudaSuccess) return;
  cudaDeviceSynchronize();
  cudaMemPoolTrimTo(pool, 0);
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// ---- launch helper ----
int Launcher::check(const char* what) {
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

int Launcher::gemm(const GemmArgs& g, bool ta, bool tb, const char* name) {
  ++*count;
  cudaError_t e = ks::gemm(g, ta, tb, st);
  if (e != cudaSuccess) return fail(KS_ERR_CUDA, "gemm %dx%dx%d: %s", g.M, g.N, g.K, cudaGetErrorString(e));
  return check(name);
}

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

// Recursive LU of columns [c0, c0+w) over rows [c0, T), pivots among rows < t_pad.
// ext > 0: the ext columns right after [c0, c0+w) (the P^T block, on the right
// spine of the recursion) take part in every merge as part of the right block,
// so U12 = L^-1 Pi P^T and the Schur block H come out of the merges' TRSMs and
// GEMMs instead of a separate TRSM chain and Schur GEMM after the LU.
// The fused TRSM+update merge (k_lu_merge, KS_FUSED_MERGE=1) is opt-in:
// measured slower than the separate trsm_ul + rlu_gemm launches at config 3.
int rlu(Launcher& L, const ks::NodeBatch& nb, int c0, int w, int pw, int* pend, int ext) {
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
  if ((h == 16 || h == 32) && w - h <= 64 && ext == 0 && L.f && L.f->knobs.fused_merge && nb.scratch) {
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

}  // namespace ksr

using namespace ksr;

extern "C" {

int ks_last_error(char* buf, int64_t len) {
  const std::string& e = last_error_msg();
  if (!buf || len <= 0) return (int)e.size();
  std::snprintf(buf, (size_t)len, "%s", e.c_str());
  return (int)e.size();
}

const char* ks_version(void) { return "libinvaskit 0.2 sm_100a (DMMA fp64, telescoping solve)"; }

int ks_trim_pool(int device) {
  KS_CUDA(cudaSetDevice(device));
  pool_trim();
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
  for (auto g : f->hst)
    if (g) cudaStreamDestroy(g);
  for (auto e : f->hfork)
    if (e) cudaEventDestroy(e);
  for (auto e : f->hjoin)
    if (e) cudaEventDestroy(e);
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
  for (auto e : f->ev_up_level)
    if (e) cudaEventDestroy(e);
  for (auto e : f->ev_up_sublev)
    if (e) cudaEventDestroy(e);
  delete f;
  if (pool_keep_gb() == 0.0) pool_trim();
}

}  // extern "C"
