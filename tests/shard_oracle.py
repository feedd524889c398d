"""CPU stand-in for one rank's sharded factor (test infrastructure).

Same methods as paper_1602_01376_b200.distributed.LibShard, computed with the
oracle's restatement of the reference formulas (oracle/ks_oracle.py) on the
rank's own subtree plus the shared top levels, so the world-size-2 gloo tests
exercise the real orchestration (factorize_sharded / solve_many_sharded) and
its NCCL-shaped exchanges without a GPU.
"""
import numpy as np
import torch

from oracle import ks_oracle as O


class OracleShard:
    def __init__(self, g: dict, shard_root: int, peers: list[int]):
        self.p = O.Problem(g)
        self.shard_root = shard_root
        self.peers = peers
        p = self.p
        lev = np.zeros(p.n_nodes, np.int64)
        for v in range(p.n_nodes):
            if not p.is_leaf(v):
                lev[p.left[v]] = lev[p.right[v]] = lev[v] + 1
        self.lev = lev
        self.k = int(lev[shard_root])
        sub, st = set(), [shard_root]
        while st:
            v = st.pop()
            sub.add(v)
            if not p.is_leaf(v):
                st += [int(p.left[v]), int(p.right[v])]
        self.sub = sub
        self.top = {v for v in range(p.n_nodes) if lev[v] < self.k}
        self.begin, self.end = int(p.begin[shard_root]), int(p.end[shard_root])
        self.s_pad = int(p.rank.max())
        self.H, self.leaf, self.node = {}, {}, {}

    def _order(self, nodes):
        return sorted(nodes, key=lambda v: (-self.lev[v], v))

    def _factor(self, nodes):
        p, n = self.p, self.p.n
        for v in self._order(nodes):
            if p.is_leaf(v):
                ids = p.node_points(v)
                A = O.kernel_block(p.coords, ids, ids, p.h) + self.lam * np.eye(ids.size)
                f = O.dense_factor(A, "cholesky")
                self.leaf[v] = f
                if p.size(v) < n:
                    P = p.coeff(v)
                    H = P @ O.dense_solve(f, P.T)
                    self.H[v] = 0.5 * (H + H.T)
                continue
            l, r = int(p.left[v]), int(p.right[v])
            B = O.kernel_block(p.coords, p.skel(l), p.skel(r), p.h)
            sl, sr = B.shape
            W = np.zeros((sl + sr, sl + sr))
            W[:sl, sl:], W[sl:, :sl] = B, B.T
            G = np.zeros_like(W)
            G[:sl, :sl], G[sl:, sl:] = self.H[l], self.H[r]
            Z = np.eye(sl + sr) + W @ G
            Zf = O.dense_factor(Z, "lu-partial-pivot")
            self.node[v] = (sl, W, G, Zf)
            if p.size(v) < n:
                P = p.coeff(v)
                M = O.solve_transposed(Zf, G).T
                M = M + O.solve_transposed(Zf, (G - M @ Z).T).T
                H = P @ M @ P.T
                self.H[v] = 0.5 * (H + H.T)

    def factorize(self, lam):
        self.lam = float(lam)
        self._factor(self.sub)

    def _pad(self, a, rows, cols):
        out = torch.zeros(rows, cols, dtype=torch.float64)
        out[: a.shape[0], : a.shape[1]] = torch.from_numpy(np.asarray(a))
        return out

    def export_h(self, node):
        return self._pad(self.H[node], self.s_pad, self.s_pad)

    def import_h(self, node, t):
        r = int(self.p.rank[node])
        self.H[node] = t[:r, :r].numpy().copy()

    def factorize_top(self):
        self._factor(self.top)

    def solve_up(self, B_local):
        p = self.p
        self.B = B_local.numpy()
        self.c, self.d = {}, {}
        for v in self._order(self.sub):
            if p.is_leaf(v):
                b = self.B[p.begin[v] - self.begin:p.end[v] - self.begin]
                self.c[v] = p.coeff(v) @ O.dense_solve(self.leaf[v], b)
            else:
                self._up_node(v)

    def _up_node(self, v):
        p = self.p
        sl, W, G, Zf = self.node[v]
        cc = np.concatenate([self.c[int(p.left[v])], self.c[int(p.right[v])]])
        rhs = W @ cc
        d = O.dense_solve(Zf, rhs)
        d = d + O.dense_solve(Zf, rhs - d - W @ (G @ d))
        self.d[v] = d
        if v != 0:
            self.c[v] = p.coeff(v) @ (cc - G @ d)

    def export_c(self, node, q):
        return self._pad(self.c[node], self.s_pad, q)

    def import_c(self, node, t):
        self.c[node] = t[: int(self.p.rank[node])].numpy().copy()

    def _down_node(self, v):
        p = self.p
        sl, W, G, Zf = self.node[v]
        u = self.d[v] if v not in self.t else O.dense_solve(Zf, p.coeff(v).T @ self.t[v]) + self.d[v]
        self.t[int(p.left[v])] = u[:sl]
        self.t[int(p.right[v])] = u[sl:]

    def solve_top(self, q):
        self.t = {}
        for v in self._order(self.top):
            self._up_node(v)
        for v in reversed(self._order(self.top)):
            self._down_node(v)

    def solve_down(self, q):
        p = self.p
        X = np.zeros_like(self.B)
        for v in reversed(self._order(self.sub)):
            if p.is_leaf(v):
                lo, hi = p.begin[v] - self.begin, p.end[v] - self.begin
                rhs = self.B[lo:hi] - (p.coeff(v).T @ self.t[v] if v in self.t else 0.0)
                X[lo:hi] = O.dense_solve(self.leaf[v], rhs)
            else:
                self._down_node(v)
        return torch.from_numpy(X)
