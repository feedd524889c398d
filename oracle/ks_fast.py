"""LAPACK-backed fast mode of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

The same algorithm as oracle/ks_oracle.py (the reference's factorize and
solve, /root/reference/pkg/src/kernelsolve/solver.py:92-237) with the
reference's in-tree Python loops replaced by LAPACK/BLAS calls that compute the
same quantities:

  leaf      A = K_leaf + lam I                       (solver.py:124, kernels.py:91-111)
            Cholesky (LAPACK potrf; the reference's _cholesky, linalg.py:185-196)
            H = sym(P A^-1 P^T)  (cho_solve: two triangular solves, solver.py:132-135)
  internal  Z = I + W G, LU with partial pivoting     (getrf: first max |.| pivot, as np.argmax; linalg.py:199-213)
            Hager cond1 estimate, 5 iterations        (linalg.py:282-304, same break rule)
            M = G Z^-1 plus ONE refinement step, H = sym(P M P^T)   (solver.py:154-164)
  solve     the O(N) telescoping form of solver.py:216-237 with the Z refinement
            step kept (ks_oracle.solve_many_telescoping, refine=True)

The Gaussian blocks use the difference form in row chunks (kernels.py:101-111)
with BLAS only for the factorizations, so the operator entries are the
reference's bit for bit. Leaves and nodes of a level run on a thread pool
(LAPACK releases the GIL, one BLAS thread per worker). Pinned to the
reference's golden fixtures by tests/test_oracle_golden.py (same bar as the
loop oracle); used by the full-size GPU parity checks at configs 3 and 4
(tests/fullsize_parity.py), where the loop oracle would take hours.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import scipy.linalg as sl

from .ks_oracle import COND_HARD, COND_WARN, IllConditioned, NotSPD, Problem, Singular  # noqa: F401


def kernel_block(coords, rows, cols, h):
    """kernels.py:91-111, difference form; chunks of 64 rows keep the
    (rows x cols x d) temporary small."""
    X = coords[rows]
    Y = coords[cols]
    out = np.empty((X.shape[0], Y.shape[0]))
    for lo in range(0, X.shape[0], 64):
        diff = X[lo:lo + 64, None, :] - Y[None, :, :]
        sq = np.einsum("ijd,ijd->ij", diff, diff)
        out[lo:lo + 64] = np.exp(sq / (-2.0 * h * h))
    return out


class LUF:
    """An LU factor of Z (LAPACK getrf) with the reference's solve API."""

    def __init__(self, Z):
        self.n = Z.shape[0]
        self.norm1 = float(np.abs(Z).sum(axis=0).max()) if self.n else 0.0
        self.lu, self.piv = sl.lu_factor(Z, check_finite=False)
        d = np.abs(np.diag(self.lu))
        if self.n and d.min() == 0.0:
            k = int(np.argmin(d))
            raise Singular(f"zero pivot column at elimination step {k}")

    def solve(self, B):
        return sl.lu_solve((self.lu, self.piv), B, trans=0, check_finite=False)

    def solve_t(self, B):
        return sl.lu_solve((self.lu, self.piv), B, trans=1, check_finite=False)


def cond1_estimate(f: LUF, max_iter: int = 5) -> float:  # linalg.py:282-304
    n = f.n
    if n == 0:
        return 0.0
    if n == 1:
        return 1.0 if f.lu[0, 0] != 0 else np.inf
    x = np.full(n, 1.0 / n)
    est = 0.0
    for _ in range(max_iter):
        y = f.solve(x)
        est = float(np.abs(y).sum())
        xi = np.where(y >= 0.0, 1.0, -1.0)
        z = f.solve_t(xi)
        j = int(np.argmax(np.abs(z)))
        if np.abs(z[j]) <= float(z @ x):
            break
        x = np.zeros(n)
        x[j] = 1.0
    if not np.isfinite(est):
        return np.inf
    return f.norm1 * est


class FastFactor:
    def __init__(self, prob: Problem, lam: float):
        self.prob = prob
        self.lam = lam
        self.leaf = {}      # node -> (cholesky lower factor, cho tuple)
        self.node = {}      # node -> (s_l, B, Hl, Hr, LUF, cond)
        self.reduced = {}   # node -> H
        self.cond = {}


def _workers() -> int:
    return int(os.environ.get("KS_ORACLE_THREADS", os.cpu_count() or 1))


def factorize(prob: Problem, lam: float) -> FastFactor:
    from threadpoolctl import threadpool_limits

    lam = float(lam)
    if not np.isfinite(lam) or lam < 0.0:  # solver.py:101-103
        raise ValueError(f"need lambda >= 0 and finite, got {lam}")
    ff = FastFactor(prob, lam)
    n = prob.n

    def leaf(v):
        ids = prob.node_points(v)
        A = kernel_block(prob.coords, ids, ids, prob.h)
        A[np.diag_indices_from(A)] += lam
        try:
            c = sl.cho_factor(A, lower=True, check_finite=False)
        except np.linalg.LinAlgError as exc:
            raise NotSPD(str(exc)) from exc
        H = None
        if prob.size(v) < n:
            P = prob.coeff(v)
            H = P @ sl.cho_solve(c, P.T, check_finite=False)
            H = 0.5 * (H + H.T)
        return v, c, H

    def internal(v):
        l, r = int(prob.left[v]), int(prob.right[v])
        B = kernel_block(prob.coords, prob.skel(l), prob.skel(r), prob.h)
        s_l, s_r = B.shape
        t = s_l + s_r
        Hl, Hr = ff.reduced[l], ff.reduced[r]
        Z = np.eye(t)
        Z[:s_l, s_l:] = B @ Hr       # (W G) with W's zero blocks skipped: same entries
        Z[s_l:, :s_l] = B.T @ Hl
        f = LUF(Z)
        cond = cond1_estimate(f)
        H = None
        if prob.size(v) < n:
            G = np.zeros((t, t))
            G[:s_l, :s_l] = Hl
            G[s_l:, s_l:] = Hr
            P = prob.coeff(v)
            M = f.solve_t(G).T                  # G Z^-1 via Z^-T G (solver.py:160)
            M = M + f.solve_t((G - M @ Z).T).T  # one refinement step (solver.py:161)
            H = P @ M @ P.T
            H = 0.5 * (H + H.T)
        return v, (s_l, B, f, cond), H

    with threadpool_limits(1), ThreadPoolExecutor(_workers()) as pool:
        for level in prob.levels_bottom_up():
            leaves = [v for v in level if prob.is_leaf(v)]
            nodes = [v for v in level if not prob.is_leaf(v)]
            for v, c, H in pool.map(leaf, leaves):
                ff.leaf[v] = c
                if H is not None:
                    ff.reduced[v] = H
            for v, nf, H in pool.map(internal, nodes):
                ff.node[v] = nf
                ff.cond[v] = nf[3]
                if H is not None:
                    ff.reduced[v] = H
            for v in sorted(nodes):  # solver.py:150-152, first failing node in processing order
                if ff.cond[v] > COND_HARD:
                    raise IllConditioned(v, ff.cond[v])
    return ff


def solve_many(ff: FastFactor, B: np.ndarray) -> np.ndarray:
    """O(N) telescoping solve with the Z refinement (ks_oracle.solve_many_telescoping)."""
    from threadpoolctl import threadpool_limits

    prob = ff.prob
    B = np.asarray(B, dtype=np.float64)
    if B.shape[1] == 0:
        return np.empty_like(B)
    if prob.is_leaf(0):
        return sl.cho_solve(ff.leaf[0], B, check_finite=False)
    c, d = {}, {}
    X = np.empty_like(B)
    with threadpool_limits(1), ThreadPoolExecutor(_workers()) as pool:
        levels = prob.levels_bottom_up()
        for level in levels:
            def up(v):
                if prob.is_leaf(v):
                    y0 = sl.cho_solve(ff.leaf[v], B[prob.begin[v]:prob.end[v]], check_finite=False)
                    return v, prob.coeff(v) @ y0, None
                s_l, Bc, f, _ = ff.node[v]
                l, r = int(prob.left[v]), int(prob.right[v])
                cc = np.concatenate([c[l], c[r]])
                Hl, Hr = ff.reduced[l], ff.reduced[r]
                rhs = np.concatenate([Bc @ cc[s_l:], Bc.T @ cc[:s_l]])       # W cc
                dv = f.solve(rhs)
                Gd = np.concatenate([Hl @ dv[:s_l], Hr @ dv[s_l:]])
                WGd = np.concatenate([Bc @ Gd[s_l:], Bc.T @ Gd[:s_l]])
                dv = dv + f.solve(rhs - dv - WGd)                            # solver.py:229-234
                cv = None
                if v != 0:
                    Gd2 = np.concatenate([Hl @ dv[:s_l], Hr @ dv[s_l:]])
                    cv = prob.coeff(v) @ (cc - Gd2)
                return v, cv, dv
            for v, cv, dv in pool.map(up, level):
                if cv is not None:
                    c[v] = cv
                if dv is not None:
                    d[v] = dv
        t_in = {}
        for level in reversed(levels):
            def down(v):
                if prob.is_leaf(v):
                    rhs = B[prob.begin[v]:prob.end[v]]
                    if v in t_in:
                        rhs = rhs - prob.coeff(v).T @ t_in[v]
                    return v, sl.cho_solve(ff.leaf[v], rhs, check_finite=False), None
                s_l, _, f, _ = ff.node[v]
                u = d[v] if v not in t_in else f.solve(prob.coeff(v).T @ t_in[v]) + d[v]
                return v, None, (u[:s_l], u[s_l:])
            for v, xv, split in pool.map(down, level):
                if xv is not None:
                    X[prob.begin[v]:prob.end[v]] = xv
                else:
                    t_in[int(prob.left[v])], t_in[int(prob.right[v])] = split
    return X


def diagnostics(ff: FastFactor) -> dict:
    zc = dict(sorted(ff.cond.items()))
    return {"z_cond": zc, "warnings": [v for v, cnd in zc.items() if cnd > COND_WARN]}
