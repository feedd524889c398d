// Persistence of operator inputs and factors in the KSINVASK container
// (container.h). The reference persists only points (points.py:65-129,
// restated in paper_1602_01376_b200/persist.py); these cache the compression
// output and the factorization across runs.
#include <type_traits>

#include "container.h"
#include "handle.h"

using namespace ksr;

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
  if (!rc) rc = save_dev(w, "xy", f->xy, sp);
  if (!rc) rc = save_dev(w, "phl", f->phl, sp);
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
  if (!rc) rc = load_dev(r, "xy", f->xy, sp);
  if (!rc) rc = load_dev(r, "phl", f->phl, sp);
  if (!rc) rc = load_dev(r, "piv", f->piv, sp);
  if (!rc) rc = load_dev(r, "pm", f->pm, sp);
  if (!rc) rc = load_dev(r, "norm1", f->norm1, sp);
  if (!rc) rc = load_dev(r, "cond", f->cond, sp);
  if (!rc) rc = load_dev(r, "leaf_info", f->leaf_info, sp);
  if (!rc) rc = load_dev(r, "int_info", f->int_info, sp);
  for (int li : fbl)
    if (li < 0 || li >= (int)f->leaf_nodes.size()) return bad(fail(KS_ERR_IO, "%s: bad fallback leaf index", path));
  if (f->int_info_h.size() != (size_t)f->n_int || f->cond_h.size() != (size_t)f->n_int ||
      f->leaf_info_h.size() != f->leaf_nodes.size())
    return bad(fail(KS_ERR_IO, "%s: diagnostics do not match the operator", path));
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


}  // extern "C"
