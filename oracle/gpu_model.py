"""Numpy model of the GPU FORMULATION — test infrastructure only.

The CUDA path does not mirror the reference's operation sequence; it computes
the same quantities through augmented factorizations:

  leaf   : Cholesky of the (m+s) x m trapezoid [[A], [P]] with A = K_leaf+lam*I
           gives L (m x m) and L21 = P L^-T;  H = L21 L21^T  (= P A^-1 P^T,
           solver.py:132-135).
  node   : LU with partial pivoting restricted to the first t rows of
              [[Z,    P^T],
               [-P G, 0  ]]      Z = I + W G  (solver.py:142-149)
           for t elimination steps; the trailing s x s block is the Schur
           complement P G Z^-1 P^T = H (solver.py:154-164).
  solve  : up   leaf z = L^-1 b, c = L21 z;  node y = L^-1 Pi (W cc),
                c = P cc + L21aug y
           down node u = U^-1 (U12aug t + y);  leaf x = L^-T (z - L21^T t)

This module checks that algebra against the oracle at small sizes, so the
CUDA kernels only have to get the block arithmetic right.
"""

from __future__ import annotations

import numpy as np

from .ks_oracle import Problem, kernel_block


def _lu_restricted(M, t):
    """Right-looking LU, t steps, pivots searched in rows [k, t) only."""
    A = M.copy()
    piv = np.arange(t)
    for k in range(t):
        p = k + int(np.argmax(np.abs(A[k:t, k])))
        piv[k] = p
        if p != k:
            A[[k, p]] = A[[p, k]]
        A[k + 1:, k] /= A[k, k]
        A[k + 1:, k + 1:] -= np.outer(A[k + 1:, k], A[k, k + 1:])
    return A, piv


def factorize_model(prob: Problem, lam: float):
    n = prob.n
    F = {"leaf": {}, "node": {}, "H": {}}
    for level_nodes in prob.levels_bottom_up():
        for v in level_nodes:
            if prob.is_leaf(v):
                ids = prob.node_points(v)
                m = ids.size
                A = kernel_block(prob.coords, ids, ids, prob.h) + lam * np.eye(m)
                s = int(prob.rank[v]) if prob.size(v) < n else 0
                T = np.vstack([A, prob.coeff(v)]) if s else A
                L = np.linalg.cholesky(A)
                L21 = np.linalg.solve(L, T[m:].T).T if s else np.zeros((0, m))
                F["leaf"][v] = (L, L21)
                if s:
                    F["H"][v] = L21 @ L21.T
                continue
            l, r = int(prob.left[v]), int(prob.right[v])
            s_l, s_r = int(prob.rank[l]), int(prob.rank[r])
            t = s_l + s_r
            B = kernel_block(prob.coords, prob.skel(l), prob.skel(r), prob.h)
            Hl, Hr = F["H"][l], F["H"][r]
            Z = np.eye(t)
            Z[:s_l, s_l:] = B @ Hr
            Z[s_l:, :s_l] = B.T @ Hl
            s = int(prob.rank[v]) if prob.size(v) < n else 0
            Aug = np.zeros((t + s, t + s))
            Aug[:t, :t] = Z
            if s:
                P = prob.coeff(v)
                Aug[:t, t:] = P.T
                Aug[t:, :s_l] = -P[:, :s_l] @ Hl
                Aug[t:, s_l:t] = -P[:, s_l:] @ Hr
            LU, piv = _lu_restricted(Aug, t)
            F["node"][v] = (LU, piv, B, t, s_l)
            if s:
                H = LU[t:, t:]
                F["H"][v] = 0.5 * (H + H.T)
    return F


def _apply_piv(piv, x):
    x = x.copy()
    for k, p in enumerate(piv):
        if p != k:
            x[[k, p]] = x[[p, k]]
    return x


def solve_model(prob: Problem, F, B):
    if prob.is_leaf(0):
        L, _ = F["leaf"][0]
        return np.linalg.solve(L.T, np.linalg.solve(L, B))
    c, y, z = {}, {}, {}
    for level_nodes in prob.levels_bottom_up():
        for v in level_nodes:
            if prob.is_leaf(v):
                L, L21 = F["leaf"][v]
                z[v] = np.linalg.solve(L, B[prob.begin[v]:prob.end[v]])
                c[v] = L21 @ z[v]
                continue
            LU, piv, Bc, t, s_l = F["node"][v]
            l, r = int(prob.left[v]), int(prob.right[v])
            cc = np.concatenate([c[l], c[r]])
            w = np.concatenate([Bc @ c[r], Bc.T @ c[l]])
            Lu = np.tril(LU[:t, :t], -1) + np.eye(t)
            y[v] = np.linalg.solve(Lu, _apply_piv(piv, w))
            if LU.shape[0] > t:
                c[v] = prob.coeff(v) @ cc + LU[t:, :t] @ y[v]
    X = np.empty_like(B)
    t_in = {}
    for level_nodes in reversed(prob.levels_bottom_up()):
        for v in level_nodes:
            if prob.is_leaf(v):
                L, L21 = F["leaf"][v]
                rhs = z[v] - (L21.T @ t_in[v] if v in t_in else 0.0)
                X[prob.begin[v]:prob.end[v]] = np.linalg.solve(L.T, rhs)
                continue
            LU, piv, Bc, t, s_l = F["node"][v]
            U = np.triu(LU[:t, :t])
            rhs = y[v] + (LU[:t, t:] @ t_in[v] if v in t_in else 0.0)
            u = np.linalg.solve(U, rhs)
            t_in[int(prob.left[v])] = u[:s_l]
            t_in[int(prob.right[v])] = u[s_l:]
    return X
