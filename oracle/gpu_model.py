"""Numpy model of the GPU FORMULATION — test infrastructure only.

The CUDA path does not mirror the reference's operation sequence; it computes
the same quantities through augmented factorizations:

  leaf   : Cholesky of the (m+s) x m trapezoid [[A], [P]] with A = K_leaf+lam*I
           gives L (m x m) and L21 = P L^-T;  H = L21 L21^T  (= P A^-1 P^T,
           solver.py:132-135).
  node   : Z = I + W G = [[I, X], [Y, I]], X = B H_r, Y = B^T H_l, eliminated
           with its identity (1,1) block as pivot: only S = I - Y X is LU-
           factored with partial pivoting, as the first s_r columns of
              [[S, E],     E = P_r^T - Y P_l^T
               [F, C]]     F = P_l H_l X - P_r H_r = -E^T H_r,  C = P_l H_l P_l^T
           (pivots among S's rows); the trailing block is C - F S^-1 E =
           P G Z^-1 P^T = H (solver.py:154-164).
  solve  : up   leaf z = L^-1 b, c = L21 z;
                node r1 = B c_r, y2 = L^-1 Pi (B^T c_l - Y r1),
                c = P cc - P_l H_l r1 + L21 y2
           down node w2 = U^-1 (y2 + U12 t), w1 = r1 + P_l^T t - X w2;
                leaf x = L^-T (z - L21^T t)

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
            B = kernel_block(prob.coords, prob.skel(l), prob.skel(r), prob.h)
            Hl, Hr = F["H"][l], F["H"][r]
            X, Y = B @ Hr, B.T @ Hl
            s = int(prob.rank[v]) if prob.size(v) < n else 0
            P = prob.coeff(v) if s else np.zeros((0, s_l + s_r))
            Pl, Pr = P[:, :s_l], P[:, s_l:]
            PHl = Pl @ Hl
            Aug = np.zeros((s_r + s, s_r + s))
            Aug[:s_r, :s_r] = np.eye(s_r) - Y @ X
            Aug[:s_r, s_r:] = Pr.T - Y @ Pl.T
            Aug[s_r:, :s_r] = -Aug[:s_r, s_r:].T @ Hr  # = P_l H_l X - P_r H_r (H symmetric): one product
            Aug[s_r:, s_r:] = PHl @ Pl.T
            LU, piv = _lu_restricted(Aug, s_r)
            F["node"][v] = (LU, piv, B, X, Y, PHl, s_l, s_r)
            if s:
                H = LU[s_r:, s_r:]
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
    c, r1s, y2s, z = {}, {}, {}, {}
    for level_nodes in prob.levels_bottom_up():
        for v in level_nodes:
            if prob.is_leaf(v):
                L, L21 = F["leaf"][v]
                z[v] = np.linalg.solve(L, B[prob.begin[v]:prob.end[v]])
                c[v] = L21 @ z[v]
                continue
            LU, piv, Bc, X, Y, PHl, s_l, s_r = F["node"][v]
            l, r = int(prob.left[v]), int(prob.right[v])
            r1 = Bc @ c[r]
            r2 = Bc.T @ c[l] - Y @ r1
            Lu = np.tril(LU[:s_r, :s_r], -1) + np.eye(s_r)
            y2 = np.linalg.solve(Lu, _apply_piv(piv, r2))
            r1s[v], y2s[v] = r1, y2
            if LU.shape[0] > s_r:
                c[v] = prob.coeff(v) @ np.concatenate([c[l], c[r]]) - PHl @ r1 + LU[s_r:, :s_r] @ y2
    X_out = np.empty_like(B)
    t_in = {}
    for level_nodes in reversed(prob.levels_bottom_up()):
        for v in level_nodes:
            if prob.is_leaf(v):
                L, L21 = F["leaf"][v]
                rhs = z[v] - (L21.T @ t_in[v] if v in t_in else 0.0)
                X_out[prob.begin[v]:prob.end[v]] = np.linalg.solve(L.T, rhs)
                continue
            LU, piv, Bc, X, Y, PHl, s_l, s_r = F["node"][v]
            y2, a1 = y2s[v].copy(), r1s[v].copy()
            if v in t_in:
                y2 = y2 + LU[:s_r, s_r:] @ t_in[v]
                a1 = a1 + prob.coeff(v)[:, :s_l].T @ t_in[v]
            w2 = np.linalg.solve(np.triu(LU[:s_r, :s_r]), y2)
            t_in[int(prob.left[v])] = a1 - X @ w2
            t_in[int(prob.right[v])] = w2
    return X_out
