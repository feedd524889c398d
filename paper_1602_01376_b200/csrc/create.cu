// ks_create / ks_create_shard: validate the reference's problem arrays, plan
// the levels (BFS levels, deepest first; subtree pipelining; padded shapes),
// allocate the handle's device buffers and start the asynchronous uploads in
// the order the first factorization consumes them.
#include <thread>

#include "handle.h"

using namespace ksr;

namespace ksr {

int create_impl(const ks_problem* p, int device, int64_t shard_root, ks_factor** out) {
  const double t_start = host_ms();
  if (!p || !out) return fail(KS_ERR_INVALID, "null argument");
  *out = nullptr;
  if (p->n < 1 || p->d < 1 || p->n_nodes < 1) return fail(KS_ERR_INVALID, "empty problem");
  if (!(p->bandwidth > 0.0) || !std::isfinite(p->bandwidth))
    return fail(KS_ERR_INVALID, "gaussian kernel needs bandwidth > 0, got %g", p->bandwidth);
  KS_CUDA(cudaSetDevice(device));
  ks_factor* f = new ks_factor();
  f->knobs = read_knobs();
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
      if (c % G || c / G < f->knobs.pipe_min) break;
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
  f->t_pad = f->s_pad;     // node LU view: pivots among S = I - Y X's rows (kernels.cuh NodeBatch)
  f->T = 2 * f->s_pad;
  f->zt = 2 * f->s_pad;
  f->R = f->m_pad + f->s_pad;
  // LU panel width of the launch sequence: register panels of 16 columns (up to
  // 1024 candidate rows, 8 beyond). KS_PANEL_W=32 selects 32-column panels where
  // they fit in shared memory: two 16-column halves and their merge in one
  // launch (k_lu_panel32) -- measured slower at config 3 (69.6 vs 69.1 ms: the
  // merge then runs on one SM per node instead of a grid); 8 forces narrow panels.
  f->pw = (f->T <= 1024) ? 16 : 8;
  if (const int w = f->knobs.panel_w) {
    ks::NodeBatch probe{};
    probe.t_pad = f->t_pad;
    probe.T = f->T;
    if (w == 32 && ks::lu_panel32_ok(probe)) f->pw = 32;
    else if (w == 8) f->pw = 8;
  }
  if (f->s_pad > 1024) { delete f; return fail(KS_ERR_UNSUPPORTED, "skeleton rank %lld too large (max 1024)", (long long)s_max); }

  const double t_plan = host_ms();
  // The points and the permutation start their DMA at once (the largest fixed
  // piece before any P block; it needs no validation result): the host checks
  // below run while it is in flight, and the device gather that trusts the
  // permutation is only queued after the permutation has been verified.
  double* orig = nullptr;
  int64_t* pmd = nullptr;
  auto early_upload = [&]() -> int {
    KS_CUDA(cudaStreamCreateWithFlags(&f->upl, cudaStreamNonBlocking));
    cudaStream_t u = f->upl;
    KS_CUDA(f->coords.alloc((size_t)(p->n + f->m_pad) * p->d));
    KS_CUDA(f->xx.alloc((size_t)p->n + f->m_pad));
    KS_CUDA(pool_alloc_async(reinterpret_cast<void**>(&orig), sizeof(double) * p->n * p->d, u));
    KS_CUDA(pool_alloc_async(reinterpret_cast<void**>(&pmd), sizeof(int64_t) * p->n, u));
    KS_CUDA(cudaMemsetAsync(f->coords.p + (size_t)p->n * p->d, 0, sizeof(double) * f->m_pad * p->d, u));
    KS_CUDA(cudaMemcpyAsync(orig, p->coords, sizeof(double) * p->n * p->d, cudaMemcpyHostToDevice, u));
    KS_CUDA(cudaMemcpyAsync(pmd, p->perm, sizeof(int64_t) * p->n, cudaMemcpyHostToDevice, u));
    f->h2d_bytes += (int64_t)(sizeof(double) * p->n * p->d + sizeof(int64_t) * p->n);
    return KS_OK;
  };
  // From here on the handle owns device memory and streams: errors go through ks_destroy.
  auto abort_create = [&](int rc) {
    if (f->upl) cudaStreamSynchronize(f->upl);
    if (orig) pool_free(orig);
    if (pmd) pool_free(pmd);
    ks_destroy(f);
    return rc;
  };
  auto bad2 = [&](const char* msg) { return abort_create(fail(KS_ERR_INVALID, "%s", msg)); };
  if (int rc = early_upload()) return abort_create(rc);
  // the permutation: host worker threads (the inverse is N random writes): pass 1
  // range-checks and inverts, pass 2 confirms pos[perm[i]] == i (any duplicate fails it).
  auto parallel_for = [](int64_t n, auto&& body) {
    const int nth = (int)std::max<int64_t>(1, std::min<int64_t>(16, n / (1 << 16)));
    std::vector<std::thread> th;
    for (int t = 1; t < nth; ++t) th.emplace_back([&, t]() { body(n * t / nth, n * (t + 1) / nth); });
    body(0, n / nth);
    for (auto& x : th) x.join();
  };
  std::vector<int64_t> pos(p->n);
  std::atomic<int> perm_bad{0}, skel_bad{0};
  const size_t nl = f->leaf_nodes.size();
  const int64_t nsk = p->skel_off[nn];
  std::vector<int> sp((size_t)nsk);
  // (on a thread of its own, beside the allocations below)
  std::thread host_checks([&]() {
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
    if (perm_bad) return;
    parallel_for(nsk, [&](int64_t a, int64_t b) {
      for (int64_t i = a; i < b; ++i) {
        const int64_t id = p->skel[i];
        if (id < 0 || id >= p->n) { skel_bad = 1; return; }
        sp[i] = (int)pos[id];
      }
    });
  });
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
    KS_CUDA(f->pn.alloc((size_t)f->n_int * f->s_pad * f->zt + 1));
    KS_CUDA(f->xy.alloc((size_t)f->n_int * 2 * f->s_pad * f->s_pad + 1));
    KS_CUDA(f->phl.alloc((size_t)f->n_int * f->s_pad * f->s_pad + 1));
    KS_CUDA(f->bt.alloc((size_t)f->n_int * f->s_pad * f->s_pad + 1));
    KS_CUDA(f->pt.alloc((size_t)f->n_int * f->zt * f->s_pad + 1));
    // GEMM-form coupling where the dimension makes it worth it (2 s^2 d per node)
    f->dk = (p->d >= 32) ? (int)roundup(p->d, 2) : 0;
    if (f->dk) {
      KS_CUDA(f->xs.alloc((size_t)f->n_int * f->zt * f->dk + 1));
      KS_CUDA(f->xn.alloc((size_t)f->n_int * f->zt + 1));
    }
    KS_CUDA(f->norm1_slab.alloc(std::max(f->n_int, 1)));
    KS_CUDA(f->norm1.alloc(std::max(f->n_int, 1)));
    KS_CUDA(f->cond.alloc(std::max(f->n_int, 1)));
    KS_CUDA(f->coeff.alloc((size_t)p->coeff_off[nn]));
    KS_CUDA(cudaStreamCreateWithFlags(&f->side, cudaStreamNonBlocking));
    KS_CUDA(cudaStreamCreateWithFlags(&f->side2, cudaStreamNonBlocking));
    KS_CUDA(cudaEventCreateWithFlags(&f->ev_fork2, cudaEventDisableTiming));
    KS_CUDA(cudaEventCreateWithFlags(&f->ev_join2, cudaEventDisableTiming));
    KS_CUDA(cudaStreamCreateWithFlags(&f->cap, cudaStreamNonBlocking));
    for (auto& g : f->gst) KS_CUDA(cudaStreamCreateWithFlags(&g, cudaStreamNonBlocking));
    for (auto& g : f->hst) KS_CUDA(cudaStreamCreateWithFlags(&g, cudaStreamNonBlocking));
    for (auto& e : f->hfork) KS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : f->hjoin) KS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
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
  const int alloc_rc = alloc_all();
  host_checks.join();
  if (alloc_rc) return abort_create(alloc_rc);
  if (perm_bad) return bad2("perm is not a permutation");
  if (skel_bad) return bad2("skeleton id out of range");
  const double t_alloc = host_ms();
  // ---- asynchronous uploads on the upload stream, in the order the first
  // factorization consumes them; the point-coordinate check overlaps the DMA.
  // Points: tree order on the device (coords_tree[i] = coords[perm[i]]) + norms.
  auto start_uploads = [&]() -> int {
    KS_CUDA(cudaEventCreateWithFlags(&f->ev_up_coords, cudaEventDisableTiming));
    KS_CUDA(cudaEventCreateWithFlags(&f->ev_up_all, cudaEventDisableTiming));
    for (auto& e : f->ev_up_leaf) KS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    f->ev_up_sublev.resize((size_t)ks_factor::kLeafChunks * f->npipe);
    for (auto& e : f->ev_up_sublev) KS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    f->ev_up_level.resize(f->levels.size());
    for (auto& e : f->ev_up_level) KS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cudaStream_t u = f->upl;
    // the small tables first (pageable sources: staged before the call returns)
    auto put = [&](auto& buf, const auto& v) -> int {
      if (!v.empty()) KS_CUDA(cudaMemcpyAsync(buf.p, v.data(), v.size() * sizeof(v[0]), cudaMemcpyHostToDevice, u));
      f->h2d_bytes += (int64_t)(v.size() * sizeof(v[0]));
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
    // the points (in flight since early_upload) to tree order, and their norms
    ks::launch_gather_rows(orig, pmd, p->n, p->d, f->coords.p, u);
    ks::launch_row_sqnorms(f->coords.p, p->n + f->m_pad, p->d, f->xx.p, u);
    KS_CUDA(cudaFreeAsync(orig, u));
    orig = nullptr;
    KS_CUDA(cudaFreeAsync(pmd, u));
    pmd = nullptr;
    KS_CUDA(cudaEventRecord(f->ev_up_coords, u));
    // P blocks: leaves in leaf order (a milestone event per leaf quarter), then
    // internal nodes level by level, deepest first (an event per level), then
    // whatever this handle does not factor; contiguous ranges are coalesced
    std::vector<char> sent(nn, 0);
    int64_t r0 = -1, r1 = -1;
    auto flush = [&]() -> int {
      if (r1 > r0) KS_CUDA(cudaMemcpyAsync(f->coeff.p + r0, p->coeff + r0, sizeof(double) * (r1 - r0),
                                           cudaMemcpyHostToDevice, u));
      if (r1 > r0) f->h2d_bytes += (int64_t)(sizeof(double) * (r1 - r0));
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
    // every leaf's P first (the leaf phase is the bulk of the work: with the
    // uploads gating it, it should start everywhere as early as possible), then
    // the pipelined levels' P subtree by subtree, then the remaining levels
    // (measured at config 3: end-to-end factorize 83 -> 79.5 ms; the reverse
    // subtree order measured 81.5 ms)
    for (int c = 0; c < ks_factor::kLeafChunks; ++c) {
      const size_t l0 = nl * c / ks_factor::kLeafChunks, l1 = nl * (c + 1) / ks_factor::kLeafChunks;
      for (size_t li = l0; li < l1; ++li)
        if (int rc = add(f->leaf_nodes[li])) return rc;
      if (int rc = flush()) return rc;
      KS_CUDA(cudaEventRecord(f->ev_up_leaf[c], u));
    }
    for (int c = 0; c < ks_factor::kLeafChunks; ++c) {
      // with subtree pipelining: this subtree's nodes of the pipelined levels
      for (int lev = 0; lev < f->npipe; ++lev) {
        const auto& lv = f->levels[lev];
        const size_t c0 = lv.size() * c / ks_factor::kLeafChunks, c1 = lv.size() * (c + 1) / ks_factor::kLeafChunks;
        for (size_t i = c0; i < c1; ++i)
          if (int rc = add(lv[i])) return rc;
        if (int rc = flush()) return rc;  // a milestone per subtree and level
        KS_CUDA(cudaEventRecord(f->ev_up_sublev[(size_t)c * f->npipe + lev], u));
      }
    }
    for (size_t lev = 0; lev < f->levels.size(); ++lev) {
      for (int v : f->levels[lev])
        if (!sent[v])
          if (int rc = add(v)) return rc;
      if (int rc = flush()) return rc;
      KS_CUDA(cudaEventRecord(f->ev_up_level[lev], u));
    }
    // a shard never reads the P of the other shards' subtrees (their H and c
    // arrive through ks_node_exchange): only its own subtree and the top levels
    for (int64_t v = 0; v < nn; ++v)
      if (!sent[v] && (in_sub[v] || f->level[v] < f->shard_level))
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

}  // namespace ksr

extern "C" {

int ks_create(const ks_problem* p, int device, ks_factor** out) { return create_impl(p, device, 0, out); }

int ks_create_shard(const ks_problem* p, int device, int64_t shard_root, ks_factor** out) {
  return create_impl(p, device, shard_root, out);
}

}  // extern "C"
