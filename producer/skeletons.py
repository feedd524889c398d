"""Batched GPU restatement of the reference skeletonization, for producing
full-size operators on the GPU box (the reference package is absent there and
its pure-Python compression would take hours at N = 1M).

Per node, bottom-up, level by level (compress.py:196-228, 285-287):
  cand  = the leaf's points (perm order) or [skel_l; skel_r]   (compress.py:206-213)
  rows  = exterior sample of max(2 s, 4 kappa) ids              (compress.py:65-69)
  block = K(rows, cand)                                         (kernels.py:73-111)
  ID    = column-pivoted Householder QR truncated at tol*|R00| or s, with the
          norm-downdate recompute guard (linalg.py:39-105);
          coeff[:, piv[:r]] = I, coeff[:, piv[r:]] = R11^-1 R12.
Rows are neighbor-guided as in the reference (producer.knn: GPU kNN restating
tree.py:146-172, sample_rows restating compress.py:145-193), or a seeded
uniform exterior draw with sampling="uniform". Operator parity with the
reference is pinned separately on the golden fixtures, where the reference's
own skeletons are used.
"""

from __future__ import annotations

import numpy as np
import torch

_NORM_GUARD = 0.01  # linalg.py:20


def _gauss(X: torch.Tensor, Y: torch.Tensor, h: float) -> torch.Tensor:
    # X (B, m, d), Y (B, n, d) -> (B, m, n), GEMM-form squared distances
    xx = (X * X).sum(-1)
    yy = (Y * Y).sum(-1)
    sq = xx[:, :, None] + yy[:, None, :] - 2.0 * torch.bmm(X, Y.transpose(1, 2))
    sq.clamp_(min=0.0)
    return torch.exp(sq / (-2.0 * h * h))


def _cpqr_id(A: torch.Tensor, tol: float, max_rank: int):
    """Batched pivoted_qr_id (linalg.py:39-105) on A (B, m, n)."""
    B, m, n = A.shape
    R = A.clone()
    ar = torch.arange(B, device=A.device)
    piv = torch.arange(n, device=A.device).repeat(B, 1)
    norms = torch.linalg.vector_norm(R, dim=1) ** 2
    ref = norms.clone()
    limit = min(max_rank, m, n)
    diag = torch.zeros(B, limit, dtype=A.dtype, device=A.device)
    for k in range(limit):
        j = k + torch.argmax(norms[:, k:], dim=1)
        # swap columns k <-> j (R, piv, norms, ref)
        ck = R[ar, :, k].clone()
        R[ar, :, k] = R[ar, :, j]
        R[ar, :, j] = ck
        for t in (piv, norms, ref):
            tk = t[ar, k].clone()
            t[ar, k] = t[ar, j]
            t[ar, j] = tk
        x = R[:, k:, k]
        normx = torch.linalg.vector_norm(x, dim=1)
        diag[:, k] = normx
        sign = torch.where(x[:, 0] >= 0, 1.0, -1.0).to(A.dtype)
        v = x.clone()
        v[:, 0] += sign * normx
        vv = (v * v).sum(1)
        beta = torch.where(vv > 0, 2.0 / torch.where(vv > 0, vv, torch.ones_like(vv)), torch.zeros_like(vv))
        blk = R[:, k:, k:]
        w = torch.bmm(v[:, None, :], blk)  # (B, 1, n-k)
        blk.baddbmm_((beta[:, None] * v)[:, :, None], w, alpha=-1.0)
        R[:, k, k] = -sign * normx
        R[:, k + 1:, k] = 0.0
        if k + 1 < n:
            norms[:, k + 1:] -= R[:, k, k + 1:] ** 2
            norms[:, k + 1:].clamp_(min=0.0)
            stale = norms[:, k + 1:] < _NORM_GUARD * ref[:, k + 1:]
            if bool(stale.any()):
                fresh = torch.linalg.vector_norm(R[:, k + 1:, k + 1:], dim=1) ** 2
                norms[:, k + 1:] = torch.where(stale, fresh, norms[:, k + 1:])
                ref[:, k + 1:] = torch.where(stale, fresh, ref[:, k + 1:])
    # rank: first k >= 1 with |R_kk| <= tol |R_00| (linalg.py:74-80)
    below = diag[:, 1:] <= tol * diag[:, :1]
    has = below.any(dim=1)
    first = torch.argmax(below.to(torch.int8), dim=1) + 1
    rank = torch.where(has, first, torch.full_like(first, limit))
    return R, piv, rank


def skeletonize(coords: np.ndarray, tree: dict, h: float, max_rank: int, tol: float = 1e-5,
                n_neighbors: int = 32, seed: int = 0, device: str = "cuda", sampling: str = "knn") -> dict:
    n, d = coords.shape
    perm = tree["perm"]
    begin, end = tree["node_begin"], tree["node_end"]
    left, right, level = tree["node_left"], tree["node_right"], tree["node_level"]
    nn = begin.size
    X = torch.from_numpy(np.ascontiguousarray(coords)).to(device)
    perm_t = torch.from_numpy(perm).to(device)
    ns = max(2 * max_rank, 4 * n_neighbors)  # compress.py:65-69
    skel: list = [None] * nn
    coeff: list = [None] * nn
    gen = torch.Generator(device=device)
    depth = int(level.max()) + 1
    if sampling == "knn":
        from .knn import knn, sample_rows
        kappa = min(n_neighbors, n - 1)
        nbr, dist = knn(X, kappa)
        pos_t = torch.empty(n, dtype=torch.int64, device=device)
        pos_t[perm_t] = torch.arange(n, device=device)
    for lev in range(depth - 1, 0, -1):  # the root has no skeleton
        nodes = [v for v in range(nn) if level[v] == lev]
        groups: dict = {}
        for v in nodes:
            nc = int(end[v] - begin[v]) if left[v] < 0 else skel[left[v]].numel() + skel[right[v]].numel()
            groups.setdefault(nc, []).append(v)
        for nc, vs in groups.items():
            cand = torch.stack([
                perm_t[int(begin[v]):int(end[v])] if left[v] < 0 else torch.cat([skel[left[v]], skel[right[v]]])
                for v in vs])
            sizes = torch.tensor([int(end[v] - begin[v]) for v in vs], device=device)
            starts = torch.tensor([int(begin[v]) for v in vs], device=device)
            budget = min(ns, n - int(sizes.max()))
            if sampling == "knn":
                rl = []
                for v in vs:
                    rl.append(sample_rows(pos_t, perm_t, int(begin[v]), int(end[v]), nbr, dist, budget, seed, v))
                rows = torch.stack(rl)
            else:
                gen.manual_seed(seed * 1_000_003 + lev * 7919 + nc)
                r = torch.rand(len(vs), budget, generator=gen, device=device, dtype=torch.float64)
                r = (r * (n - sizes)[:, None].to(torch.float64)).long()
                pos = r + (r >= starts[:, None]).long() * sizes[:, None]
                rows = perm_t[pos]
            A = _gauss(X[rows], X[cand], h)
            R, piv, rank = _cpqr_id(A, tol, max_rank)
            for rk in torch.unique(rank).tolist():
                sel = (rank == rk).nonzero().flatten()
                Rs, ps = R[sel], piv[sel]
                T = torch.linalg.solve_triangular(Rs[:, :rk, :rk], Rs[:, :rk, rk:], upper=True)
                Bs = sel.numel()
                C = torch.zeros(Bs, rk, nc, dtype=torch.float64, device=device)
                eye = torch.eye(rk, dtype=torch.float64, device=device).expand(Bs, rk, rk)
                C.scatter_(2, ps[:, None, :rk].expand(Bs, rk, rk), eye)
                C.scatter_(2, ps[:, None, rk:].expand(Bs, rk, nc - rk), T)
                sk = torch.gather(cand[sel], 1, ps[:, :rk])
                for i, b in enumerate(sel.tolist()):
                    v = vs[b]
                    skel[v] = sk[i]
                    coeff[v] = C[i]
    rank_arr = np.zeros(nn, np.int64)
    skel_off = np.zeros(nn + 1, np.int64)
    coeff_off = np.zeros(nn + 1, np.int64)
    for v in range(nn):
        if skel[v] is not None:
            rank_arr[v] = skel[v].numel()
        skel_off[v + 1] = skel_off[v] + rank_arr[v]
        coeff_off[v + 1] = coeff_off[v] + (coeff[v].numel() if coeff[v] is not None else 0)
    skel_all = torch.cat([s for s in skel if s is not None]).cpu().numpy() if nn > 1 else np.zeros(0, np.int64)
    coeff_all = np.empty(int(coeff_off[-1]), np.float64)
    # stream P blocks to the host level by level (keeps device memory bounded)
    for v in range(nn):
        if coeff[v] is not None:
            coeff_all[coeff_off[v]:coeff_off[v + 1]] = coeff[v].reshape(-1).cpu().numpy()
    return {"rank": rank_arr, "skel_off": skel_off, "skel": skel_all.astype(np.int64),
            "coeff_off": coeff_off, "coeff": coeff_all}
