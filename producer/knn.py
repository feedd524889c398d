"""GPU k-nearest neighbors and neighbor-guided row sampling for the operator
producer (restating tree.py:146-172 and compress.py:145-193).

kNN: fp32 GEMM-form distances pick 8 extra candidates per point, which are
re-ranked with fp64 squared distances in the reference's expression
(||x||^2 + ||y||^2 - 2 x.y, clipped at 0, self excluded, ties to the smaller
id). Near-ties at the fp32 resolution can order differently from the
reference's fp64 sweep; the producer only needs the same construction, not
bit-identical lists (parity is pinned on the reference's own operators).
"""

from __future__ import annotations

import numpy as np
import torch


def knn(X: torch.Tensor, k: int, chunk: int = 1024, extra: int = 8):
    """(nbr int64 (n, k), dist float64 (n, k)) on X's device."""
    n = X.shape[0]
    xx = (X * X).sum(1)
    X32 = X.float()
    xx32 = xx.float()
    nbr = torch.empty(n, k, dtype=torch.int64, device=X.device)
    dist = torch.empty(n, k, dtype=torch.float64, device=X.device)
    kk = min(n - 1, k + extra)
    for lo in range(0, n, chunk):
        hi = min(lo + chunk, n)
        rows = torch.arange(lo, hi, device=X.device)
        d32 = xx32[lo:hi, None] + xx32[None, :] - 2.0 * (X32[lo:hi] @ X32.T)
        d32[torch.arange(hi - lo, device=X.device), rows] = float("inf")
        cand = torch.topk(d32, kk + 1, dim=1, largest=False).indices  # (c, kk+1)
        del d32
        sq = xx[lo:hi, None] + xx[cand] - 2.0 * torch.einsum("cd,ckd->ck", X[lo:hi], X[cand])
        sq.clamp_(min=0.0)
        sq[cand == rows[:, None]] = float("inf")
        # order by (sq, id): stable sort by id, then stable sort by sq
        o1 = torch.argsort(cand, dim=1, stable=True)
        cand, sq = torch.gather(cand, 1, o1), torch.gather(sq, 1, o1)
        o2 = torch.argsort(sq, dim=1, stable=True)
        cand, sq = torch.gather(cand, 1, o2), torch.gather(sq, 1, o2)
        nbr[lo:hi] = cand[:, :k]
        dist[lo:hi] = torch.sqrt(sq[:, :k])
    return nbr, dist


def sample_rows(pos: torch.Tensor, perm: torch.Tensor, begin: int, end: int, nbr: torch.Tensor,
                dist: torch.Tensor, n_samples: int, seed: int, node_id: int) -> torch.Tensor:
    """compress.py:145-193 for one node: exterior neighbors of the node's points,
    ordered by distance (ties to the smaller id), deduplicated keeping the first
    occurrence, cut at min(n_samples, n - size); the fill-up is the reference's
    own draw, generator(seed, 0x726F77, node_id).choice(pool, need, replace=False)
    over the ascending exterior pool (compress.py:185-191), on the host."""
    from paper_1602_01376_b200.rng import generator
    n = perm.numel()
    size = end - begin
    budget = min(n_samples, n - size)
    owned = perm[begin:end]
    cid = nbr[owned].reshape(-1)
    cd = dist[owned].reshape(-1)
    p = pos[cid]
    keep = (p < begin) | (p >= end)
    cid, cd = cid[keep], cd[keep]
    if cid.numel():
        o1 = torch.argsort(cid, stable=True)
        cid, cd = cid[o1], cd[o1]
        o2 = torch.argsort(cd, stable=True)
        cid = cid[o2]
        # first occurrence of each id in this order
        order = torch.arange(cid.numel(), device=cid.device)
        u, inv = torch.unique(cid, return_inverse=True)
        first = torch.full((u.numel(),), cid.numel(), dtype=torch.int64, device=cid.device)
        first.scatter_reduce_(0, inv, order, reduce="amin")
        chosen = cid[torch.sort(first).values][:budget]
    else:
        chosen = cid[:0]
    need = budget - chosen.numel()
    if need > 0:
        pool_mask = torch.ones(n, dtype=torch.bool, device=perm.device)
        pool_mask[owned] = False
        pool_mask[chosen] = False
        pool = torch.nonzero(pool_mask).flatten().cpu().numpy()
        extra = generator(seed, 0x726F77, node_id).choice(pool, size=need, replace=False)
        chosen = torch.cat([chosen, torch.from_numpy(extra.astype(np.int64)).to(perm.device)])
    return chosen
