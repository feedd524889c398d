// Diagnostics (HierFactor.diagnostics, solver.py:111-116,175-188), debug views
// of the factor (parity debugging), profiling, the GEMM test hooks, and the
// dense cross-kernel matvec of krr_predict (solver.py:273-301).
#include "handle.h"

using namespace ksr;

extern "C" {

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
  const SolveWs* w = f->last_ws;  // the workspace of the last solve
  if (which <= 3 && !w) return fail(KS_ERR_INVALID, "no solve has run on this handle");
  switch (which) {
    case 0: base = w->z.p; stride = (int64_t)f->m_pad * w->q_cap; break;      // per leaf index
    case 1: base = w->c.p; stride = (int64_t)f->s_pad * w->q_cap; break;      // per node
    case 2: base = w->tin.p; stride = (int64_t)f->s_pad * w->q_cap; break;    // per node
    case 3: base = w->y.p; stride = (int64_t)f->zt * w->q_cap; break;         // per internal index
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
  const SolveWs* w = f->last_ws;
  switch (which) {
    case 0: return w ? (int64_t)w->z.p : 0;
    case 1: return w ? (int64_t)w->c.p : 0;
    case 2: return w ? (int64_t)w->tin.p : 0;
    case 3: return w ? (int64_t)w->y.p : 0;
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
  out8[4] = f->R; out8[5] = f->last_ws ? f->last_ws->q_cap : 0; out8[6] = f->n_int; out8[7] = (int64_t)f->leaf_nodes.size();
  return KS_OK;
}

int64_t ks_device_bytes(const ks_factor* f) {
  if (!f) return 0;
  int64_t b = 0;
  b += f->coords.n * 8 + f->coeff.n * 8 + f->leafA.n * 8 + f->inv.n * 8 + f->hbuf.n * 8 + f->aug.n * 8;
  b += f->bc.n * 8 + f->pn.n * 8 + f->xy.n * 8 + f->phl.n * 8;
  std::lock_guard<std::mutex> lk(const_cast<ks_factor*>(f)->ws_mu);
  for (const auto& w : f->ws)
    b += 8 * (int64_t)(w->z.n + w->c.n + w->tin.n + w->y.n + w->wtmp.n + w->bdev.n + w->xdev.n + w->fb_y.n +
                       w->mv_c.n + w->mv_inc.n + w->mv_tot.n);
  return b;
}

int64_t ks_upload_bytes(const ks_factor* f) { return f ? f->h2d_bytes : 0; }

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

int ks_pipelined_levels(const ks_factor* f, int* out2) {
  if (!f || !out2) return fail(KS_ERR_INVALID, "null argument");
  out2[0] = f->npipe;
  out2[1] = (f->npipe > 0 && f->knobs.pipe && f->knobs.groups == ks_factor::kLeafChunks) ? f->npipe : 0;
  return KS_OK;
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

}  // extern "C"
