"""CPU oracle for the Inv-ASKIT factor/solve hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference `kernelsolve` factor/solve
path (`/root/reference/pkg/src/kernelsolve/solver.py:92-237`, its dense
micro-kernels `linalg.py:116-304` and the Gaussian block `kernels.py:91-111`).
It is the checker for the CUDA path: only `tests/`, `__graft_entry__.smoke()`
and `bench.py`'s CPU-baseline leg may import it. The product package never
imports it and has no CPU fallback.

Parity is PINNED: `tests/test_oracle_golden.py` checks this restatement against
golden vectors produced by running the reference itself (`tests/golden/
make_golden.py`, committed fixtures `tests/golden/*.npz`): leaf Cholesky
factors, reduced matrices H, Z condition estimates and the solution u.

Problem format (plain arrays, shared with the fixtures and the C-ABI marshal):
  coords (n, d) ORIGINAL order; perm (n,); node_begin/end/level/left/right
  (n_nodes,), left/right = -1 at leaves; rank (n_nodes,) (0 = no skeleton);
  skel_off/skel (global ids, pivot order); coeff_off/coeff (P row-major,
  rank x |cand|); h (Gaussian bandwidth).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

COND_HARD = 1e14  # solver.py:50
COND_WARN = 1e10  # solver.py:51


class OracleError(Exception):
    pass


class NotSPD(OracleError):
    pass


class Singular(OracleError):
    pass


class IllConditioned(OracleError):
    def __init__(self, node_id, cond):
        self.node_id = node_id
        self.cond_estimate = cond
        super().__init__(f"node {node_id}: cond {cond:.3e}")


# --------------------------------------------------------------------------
# problem accessors
# --------------------------------------------------------------------------
class Problem:
    """Read-only view over the plain-array problem dict."""

    def __init__(self, arrs: dict):
        self.a = arrs
        self.coords = np.asarray(arrs["coords"], dtype=np.float64)
        self.perm = np.asarray(arrs["perm"], dtype=np.int64)
        self.begin = np.asarray(arrs["node_begin"], dtype=np.int64)
        self.end = np.asarray(arrs["node_end"], dtype=np.int64)
        self.level = np.asarray(arrs["node_level"], dtype=np.int64)
        self.left = np.asarray(arrs["node_left"], dtype=np.int64)
        self.right = np.asarray(arrs["node_right"], dtype=np.int64)
        self.rank = np.asarray(arrs["rank"], dtype=np.int64)
        self.skel_off = np.asarray(arrs["skel_off"], dtype=np.int64)
        self.skel_ids = np.asarray(arrs["skel"], dtype=np.int64)
        self.coeff_off = np.asarray(arrs["coeff_off"], dtype=np.int64)
        self.coeff_all = np.asarray(arrs["coeff"], dtype=np.float64)
        self.h = float(arrs["h"])
        self.n = self.perm.size
        self.n_nodes = self.begin.size

    def is_leaf(self, v):
        return self.left[v] < 0

    def size(self, v):
        return int(self.end[v] - self.begin[v])

    def skel(self, v):
        return self.skel_ids[self.skel_off[v]:self.skel_off[v + 1]]

    def coeff(self, v):
        r = int(self.rank[v])
        flat = self.coeff_all[self.coeff_off[v]:self.coeff_off[v + 1]]
        return flat.reshape(r, -1) if r else flat.reshape(0, 0)

    def node_points(self, v):
        # tree.py:231-234
        return self.perm[self.begin[v]:self.end[v]]

    def levels_bottom_up(self):
        # tree.py:239-244
        depth = int(self.level.max()) + 1
        by = [[] for _ in range(depth)]
        for v in range(self.n_nodes):
            by[int(self.level[v])].append(v)
        return by[::-1]


# --------------------------------------------------------------------------
# Gaussian block, kernels.py:91-111 (difference form, same einsum contraction)
# --------------------------------------------------------------------------
def kernel_block(coords, rows, cols, h):
    X = coords[rows]
    Y = coords[cols]
    out = np.empty((X.shape[0], Y.shape[0]))
    d = max(1, X.shape[1])
    chunk = max(1, (1 << 24) // max(1, Y.shape[0] * d))  # kernels.py:26,94
    for lo in range(0, X.shape[0], chunk):
        hi = min(lo + chunk, X.shape[0])
        diff = X[lo:hi, None, :] - Y[None, :, :]
        sq = np.einsum("ijd,ijd->ij", diff, diff)
        out[lo:hi] = np.exp(sq / (-2.0 * h * h))
    return out


# --------------------------------------------------------------------------
# dense micro-kernels, linalg.py:116-304
# --------------------------------------------------------------------------
@dataclass
class Factor:
    kind: str
    size: int
    norm1: float
    lower: np.ndarray | None = None
    lu: np.ndarray | None = None
    row_swaps: np.ndarray | None = None


def _solve_upper(U, B):  # linalg.py:116-124
    s = U.shape[0]
    X = np.array(B, dtype=np.float64, copy=True)
    for i in range(s - 1, -1, -1):
        if i + 1 < s:
            X[i] -= U[i, i + 1:] @ X[i + 1:]
        X[i] /= U[i, i]
    return X


def _solve_lower(L, B, unit=False):  # linalg.py:127-136
    n = L.shape[0]
    X = np.array(B, dtype=np.float64, copy=True)
    for i in range(n):
        if i > 0:
            X[i] -= L[i, :i] @ X[:i]
        if not unit:
            X[i] /= L[i, i]
    return X


def _solve_unit_upper(U, B):  # linalg.py:139-145
    n = U.shape[0]
    X = np.array(B, dtype=np.float64, copy=True)
    for i in range(n - 1, -1, -1):
        if i + 1 < n:
            X[i] -= U[i, i + 1:] @ X[i + 1:]
    return X


def _solve_upper_from_lower(L, B):  # linalg.py:235-243
    n = L.shape[0]
    X = np.array(B, dtype=np.float64, copy=True)
    for i in range(n - 1, -1, -1):
        if i + 1 < n:
            X[i] -= L[i + 1:, i] @ X[i + 1:]
        X[i] /= L[i, i]
    return X


def cholesky(A):  # linalg.py:185-196
    n = A.shape[0]
    L = np.zeros((n, n))
    for j in range(n):
        col = A[j:, j] - L[j:, :j] @ L[j, :j]
        pivot = float(col[0])
        if pivot <= 0.0 or not np.isfinite(pivot):
            raise NotSPD(f"non-positive pivot {pivot:.3e} at column {j}")
        ljj = np.sqrt(pivot)
        L[j, j] = ljj
        L[j + 1:, j] = col[1:] / ljj
    return L


def lu_partial_pivot(A):  # linalg.py:199-213
    n = A.shape[0]
    LU = A.copy()
    swaps = np.arange(n, dtype=np.int64)
    for k in range(n):
        p = k + int(np.argmax(np.abs(LU[k:, k])))
        if LU[p, k] == 0.0:
            raise Singular(f"zero pivot column at elimination step {k}")
        swaps[k] = p
        if p != k:
            LU[[k, p]] = LU[[p, k]]
        if k + 1 < n:
            LU[k + 1:, k] /= LU[k, k]
            LU[k + 1:, k + 1:] -= np.outer(LU[k + 1:, k], LU[k, k + 1:])
    return LU, swaps


def dense_factor(A, kind="cholesky"):  # linalg.py:165-182
    A = np.asarray(A, dtype=np.float64)
    n = A.shape[0]
    norm1 = float(np.abs(A).sum(axis=0).max()) if n else 0.0
    if kind == "cholesky":
        return Factor(kind, n, norm1, lower=cholesky(A))
    lu, swaps = lu_partial_pivot(A)
    return Factor(kind, n, norm1, lu=lu, row_swaps=swaps)


def _lu_solve(f, B, trans):  # linalg.py:246-263
    X = np.array(B, dtype=np.float64, copy=True)
    n = f.size
    if not trans:
        for k in range(n):
            p = f.row_swaps[k]
            if p != k:
                X[[k, p]] = X[[p, k]]
        X = _solve_lower(f.lu, X, unit=True)
        return _solve_upper(f.lu, X)
    X = _solve_lower(f.lu.T, X, unit=False)
    X = _solve_unit_upper(f.lu.T, X)
    for k in range(n - 1, -1, -1):
        p = f.row_swaps[k]
        if p != k:
            X[[k, p]] = X[[p, k]]
    return X


def dense_solve(f, B):  # linalg.py:216-232
    B = np.asarray(B, dtype=np.float64)
    vector = B.ndim == 1
    if vector:
        B = B[:, None]
    if B.shape[1] == 0:
        X = B.copy()
    elif f.kind == "cholesky":
        X = _solve_upper_from_lower(f.lower, _solve_lower(f.lower, B))
    else:
        X = _lu_solve(f, B, trans=False)
    return X[:, 0] if vector else X


def solve_transposed(f, B):  # linalg.py:266-279
    if f.kind == "cholesky":
        return dense_solve(f, B)
    B = np.asarray(B, dtype=np.float64)
    vector = B.ndim == 1
    if vector:
        B = B[:, None]
    X = _lu_solve(f, B, trans=True)
    return X[:, 0] if vector else X


def cond1_estimate(f, max_iter=5):  # linalg.py:282-304
    n = f.size
    if n == 0:
        return 0.0
    if n == 1:
        diag = f.lower[0, 0] ** 2 if f.kind == "cholesky" else f.lu[0, 0]
        return 1.0 if diag != 0 else np.inf
    x = np.full(n, 1.0 / n)
    est = 0.0
    for _ in range(max_iter):
        y = dense_solve(f, x)
        est = float(np.abs(y).sum())
        xi = np.where(y >= 0.0, 1.0, -1.0)
        z = solve_transposed(f, xi)
        j = int(np.argmax(np.abs(z)))
        if np.abs(z[j]) <= float(z @ x):
            break
        x = np.zeros(n)
        x[j] = 1.0
    if not np.isfinite(est):
        return np.inf
    return f.norm1 * est


# --------------------------------------------------------------------------
# factorize, solver.py:92-189
# --------------------------------------------------------------------------
@dataclass
class NodeF:
    s_l: int
    s_r: int
    W: np.ndarray
    G: np.ndarray
    Zf: Factor
    cond: float
    H: np.ndarray | None = None


@dataclass
class OracleFactor:
    prob: Problem
    lam: float
    leaf: dict = field(default_factory=dict)     # node -> (Factor, fallback)
    node: dict = field(default_factory=dict)     # node -> NodeF
    reduced: dict = field(default_factory=dict)  # node -> H (sym)
    diagnostics: dict = field(default_factory=dict)


def factorize(prob: Problem, lam: float) -> OracleFactor:
    lam = float(lam)
    if not np.isfinite(lam) or lam < 0.0:  # solver.py:101-103
        raise ValueError(f"need lambda >= 0 and finite, got {lam}")
    of = OracleFactor(prob, lam)
    n = prob.n
    for level_nodes in prob.levels_bottom_up():  # solver.py:167-173
        for v in level_nodes:
            if prob.is_leaf(v):  # solver.py:123-136
                ids = prob.node_points(v)
                block = kernel_block(prob.coords, ids, ids, prob.h) + lam * np.eye(ids.size)
                try:
                    f = dense_factor(block, "cholesky")
                    fb = False
                except NotSPD:
                    f = dense_factor(block, "lu-partial-pivot")
                    fb = True
                of.leaf[v] = (f, fb)
                if prob.size(v) < n:
                    P = prob.coeff(v)
                    H = P @ dense_solve(f, P.T)
                    of.reduced[v] = 0.5 * (H + H.T)
                continue
            l, r = int(prob.left[v]), int(prob.right[v])  # solver.py:138-165
            B = kernel_block(prob.coords, prob.skel(l), prob.skel(r), prob.h)
            s_l, s_r = B.shape
            m = s_l + s_r
            W = np.zeros((m, m))
            W[:s_l, s_l:] = B
            W[s_l:, :s_l] = B.T
            G = np.zeros((m, m))
            G[:s_l, :s_l] = of.reduced[l]
            G[s_l:, s_l:] = of.reduced[r]
            Z = np.eye(m) + W @ G
            Zf = dense_factor(Z, "lu-partial-pivot")
            cond = cond1_estimate(Zf)
            if cond > COND_HARD:
                raise IllConditioned(v, cond)
            nf = NodeF(s_l, s_r, W, G, Zf, cond)
            if prob.size(v) < n:
                P = prob.coeff(v)
                M = solve_transposed(Zf, G).T
                M = M + solve_transposed(Zf, (G - M @ Z).T).T
                H = P @ M @ P.T
                nf.H = 0.5 * (H + H.T)
                of.reduced[v] = nf.H
            of.node[v] = nf
    fallback = sorted(v for v, (_, fb) in of.leaf.items() if fb)
    of.diagnostics = {  # solver.py:175-188
        "cholesky_fallbacks": len(fallback),
        "fallback_nodes": fallback,
        "z_cond": {v: nf.cond for v, nf in sorted(of.node.items())},
        "warnings": [
            f"node {v}: Z condition estimate {nf.cond:.3e} exceeds {COND_WARN:.0e}; "
            f"results may lose accuracy"
            for v, nf in sorted(of.node.items()) if nf.cond > COND_WARN
        ],
    }
    return of


# --------------------------------------------------------------------------
# telescoping basis ops, compress.py:305-349
# --------------------------------------------------------------------------
def apply_prolongation(prob, v, c):
    t = prob.coeff(v).T @ c
    if prob.is_leaf(v):
        return t
    l, r = int(prob.left[v]), int(prob.right[v])
    s_l = int(prob.rank[l])
    return np.concatenate([apply_prolongation(prob, l, t[:s_l]),
                           apply_prolongation(prob, r, t[s_l:])])


def skel_project(prob, v, y):
    if prob.is_leaf(v):
        return prob.coeff(v) @ y
    l, r = int(prob.left[v]), int(prob.right[v])
    n_l = prob.size(l)
    stacked = np.concatenate([skel_project(prob, l, y[:n_l]), skel_project(prob, r, y[n_l:])])
    return prob.coeff(v) @ stacked


# --------------------------------------------------------------------------
# recursive solve, solver.py:200-237 (the reference's own O((N/m)^2) recursion)
# --------------------------------------------------------------------------
def solve_many_recursive(of: OracleFactor, B: np.ndarray) -> np.ndarray:
    B = np.asarray(B, dtype=np.float64)
    if B.shape[1] == 0:
        return np.empty_like(B)
    return _solve_node(of, 0, B)


def _solve_node(of, v, B):
    prob = of.prob
    if prob.is_leaf(v):
        return dense_solve(of.leaf[v][0], B)
    l, r = int(prob.left[v]), int(prob.right[v])
    n_l = prob.size(l)
    y_l = _solve_node(of, l, B[:n_l])
    y_r = _solve_node(of, r, B[n_l:])
    nf = of.node[v]
    c = np.concatenate([skel_project(prob, l, y_l), skel_project(prob, r, y_r)])
    rhs = nf.W @ c
    d = dense_solve(nf.Zf, rhs)
    d = d + dense_solve(nf.Zf, rhs - d - nf.W @ (nf.G @ d))
    e_l = _solve_node(of, l, apply_prolongation(prob, l, d[:nf.s_l]))
    e_r = _solve_node(of, r, apply_prolongation(prob, r, d[nf.s_l:]))
    return np.concatenate([y_l - e_l, y_r - e_r])


# --------------------------------------------------------------------------
# O(N) telescoping solve: same factors, each node visited
# once on the way up and once on the way down. Algebraically identical to
# the recursion above (refine=True keeps its Z refinement step).
# --------------------------------------------------------------------------
def solve_many_telescoping(of: OracleFactor, B: np.ndarray, refine: bool = True) -> np.ndarray:
    prob = of.prob
    B = np.asarray(B, dtype=np.float64)
    if B.shape[1] == 0:
        return np.empty_like(B)
    if prob.is_leaf(0):
        return dense_solve(of.leaf[0][0], B)
    c, d = {}, {}
    for level_nodes in prob.levels_bottom_up():
        for v in level_nodes:
            if prob.is_leaf(v):
                y0 = dense_solve(of.leaf[v][0], B[prob.begin[v]:prob.end[v]])
                c[v] = prob.coeff(v) @ y0
                continue
            l, r = int(prob.left[v]), int(prob.right[v])
            nf = of.node[v]
            cc = np.concatenate([c[l], c[r]])
            rhs = nf.W @ cc
            dv = dense_solve(nf.Zf, rhs)
            if refine:
                dv = dv + dense_solve(nf.Zf, rhs - dv - nf.W @ (nf.G @ dv))
            d[v] = (dv, cc)
            if v != 0:
                c[v] = prob.coeff(v) @ (cc - nf.G @ dv)
    X = np.empty_like(B)
    t_in = {}
    for level_nodes in reversed(prob.levels_bottom_up()):
        for v in level_nodes:
            if prob.is_leaf(v):
                rhs = B[prob.begin[v]:prob.end[v]]
                if v in t_in:
                    rhs = rhs - prob.coeff(v).T @ t_in[v]
                X[prob.begin[v]:prob.end[v]] = dense_solve(of.leaf[v][0], rhs)
                continue
            nf = of.node[v]
            dv = d[v][0]
            u = dv if v not in t_in else dense_solve(nf.Zf, prob.coeff(v).T @ t_in[v]) + dv
            t_in[int(prob.left[v])] = u[:nf.s_l]
            t_in[int(prob.right[v])] = u[nf.s_l:]
    return X


# --------------------------------------------------------------------------
# compressed matvec, compress.py:352-411 (residual checks at full sizes)
# --------------------------------------------------------------------------
def hss_matvec(prob: Problem, w: np.ndarray) -> np.ndarray:
    w = np.asarray(w, dtype=np.float64)
    if prob.is_leaf(0):
        ids = prob.node_points(0)
        return kernel_block(prob.coords, ids, ids, prob.h) @ w
    weights = {}
    for level_nodes in prob.levels_bottom_up():
        for v in level_nodes:
            if prob.rank[v] == 0:
                continue
            if prob.is_leaf(v):
                weights[v] = prob.coeff(v) @ w[prob.begin[v]:prob.end[v]]
            else:
                weights[v] = prob.coeff(v) @ np.concatenate(
                    [weights[int(prob.left[v])], weights[int(prob.right[v])]])
    incoming = {}
    for v in range(prob.n_nodes):
        if prob.is_leaf(v):
            continue
        l, r = int(prob.left[v]), int(prob.right[v])
        Bc = kernel_block(prob.coords, prob.skel(l), prob.skel(r), prob.h)
        incoming[l] = Bc @ weights[r]
        incoming[r] = Bc.T @ weights[l]
    totals = {}
    for level_nodes in reversed(prob.levels_bottom_up()):
        for v in level_nodes:
            if prob.is_leaf(v):
                continue
            l, r = int(prob.left[v]), int(prob.right[v])
            if v in totals:
                t = prob.coeff(v).T @ totals[v]
                s_l = int(prob.rank[l])
                totals[l] = incoming[l] + t[:s_l]
                totals[r] = incoming[r] + t[s_l:]
            else:
                totals[l] = incoming[l]
                totals[r] = incoming[r]
    out = np.empty_like(w)
    for v in range(prob.n_nodes):
        if not prob.is_leaf(v):
            continue
        seg = slice(prob.begin[v], prob.end[v])
        ids = prob.node_points(v)
        out[seg] = kernel_block(prob.coords, ids, ids, prob.h) @ w[seg]
        out[seg] += prob.coeff(v).T @ totals[v]
    return out


# --------------------------------------------------------------------------
# KRR front ends, solver.py:240-301
# --------------------------------------------------------------------------
def krr_weights(prob: Problem, lam: float, y: np.ndarray) -> np.ndarray:
    """krr_fit after tree + compress (solver.py:264-270): solve in tree order,
    weights back in original order."""
    of = factorize(prob, lam)
    w_perm = solve_many_telescoping(of, np.asarray(y, dtype=np.float64)[prob.perm][:, None])[:, 0]
    w = np.empty_like(w_perm)
    w[prob.perm] = w_perm
    return w


def krr_predict(x_train: np.ndarray, w: np.ndarray, h: float, x_test: np.ndarray) -> np.ndarray:
    """sum_i k(x_test_j, x_train_i) w_i, dense (solver.py:273-301): the same
    merged-point-set kernel_block over row blocks of the test set."""
    if x_test.shape[0] == 0:
        return np.empty(0)
    merged = np.vstack([x_test, x_train])
    train_cols = x_test.shape[0] + np.arange(x_train.shape[0])
    out = np.empty(x_test.shape[0])
    step = max(1, (1 << 24) // max(x_train.shape[0], 1))
    for start in range(0, x_test.shape[0], step):
        stop = min(start + step, x_test.shape[0])
        out[start:stop] = kernel_block(merged, np.arange(start, stop), train_cols, h) @ w
    return out
