"""Marshalling of the operator inputs into the C-ABI problem (include/invaskit.h).

Two sources are accepted:
  * a reference `kernelsolve.CompressedKernel` (compress.py:93-142), read
    duck-typed: `ck.points.coords`, `ck.tree.perm`, `ck.tree.nodes[*]`
    (`begin`, `end`, `children`, tree.py:27-50), `ck.skeletons[*]` (`skel`,
    `coeff`, compress.py:72-90) and `ck.spec.bandwidth` (kernels.py:29-59);
  * the plain-array problem dict used by the golden fixtures and the bench
    (keys `coords, perm, node_begin, node_end, node_left, node_right, rank,
    skel_off, skel, coeff_off, coeff, h`).
Both become the same contiguous int64/float64 arrays the library copies.
"""

from __future__ import annotations

import ctypes as C
import hashlib
from dataclasses import dataclass

import numpy as np

from ._lib import KsProblem
from .errors import InvalidArgumentError


@dataclass
class Problem:
    coords: np.ndarray      # (n, d) float64, ORIGINAL order
    perm: np.ndarray        # (n,) int64
    node_begin: np.ndarray  # (n_nodes,) int64
    node_end: np.ndarray
    node_left: np.ndarray   # -1 at leaves
    node_right: np.ndarray
    rank: np.ndarray        # 0 = no skeleton (root)
    skel_off: np.ndarray    # (n_nodes+1,)
    skel: np.ndarray        # global ids, pivot order
    coeff_off: np.ndarray   # (n_nodes+1,)
    coeff: np.ndarray       # P blocks, rank x |cand| row-major, concatenated
    h: float

    @property
    def n(self) -> int:
        return int(self.perm.size)

    @property
    def d(self) -> int:
        return int(self.coords.shape[1])

    @property
    def n_nodes(self) -> int:
        return int(self.node_begin.size)

    def int_hash(self) -> str:
        """sha256 of the integer bookkeeping (tree perm, node table, ranks,
        skeleton ids): the bit-exact part of the parity contract."""
        h = hashlib.sha256()
        for a in (self.perm, self.node_begin, self.node_end, self.node_level(), self.node_left,
                  self.node_right, self.rank, self.skel_off, self.skel):
            h.update(np.ascontiguousarray(a, dtype="<i8").tobytes())
        return h.hexdigest()

    def node_level(self) -> np.ndarray:
        lev = np.zeros(self.n_nodes, np.int64)
        for v in range(self.n_nodes):
            for c in (self.node_left[v], self.node_right[v]):
                if c >= 0:
                    lev[c] = lev[v] + 1
        return lev

    def to_c(self) -> KsProblem:
        def p64(a):
            return a.ctypes.data_as(C.POINTER(C.c_int64))

        def pf(a):
            return a.ctypes.data_as(C.POINTER(C.c_double))

        return KsProblem(
            n=self.n, d=self.d, coords=pf(self.coords), perm=p64(self.perm), n_nodes=self.n_nodes,
            node_begin=p64(self.node_begin), node_end=p64(self.node_end), node_left=p64(self.node_left),
            node_right=p64(self.node_right), rank=p64(self.rank), skel_off=p64(self.skel_off),
            skel=p64(self.skel), coeff_off=p64(self.coeff_off), coeff=pf(self.coeff), bandwidth=float(self.h))


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def from_arrays(d: dict) -> Problem:
    return Problem(
        coords=_f64(d["coords"]), perm=_i64(d["perm"]), node_begin=_i64(d["node_begin"]),
        node_end=_i64(d["node_end"]), node_left=_i64(d["node_left"]), node_right=_i64(d["node_right"]),
        rank=_i64(d["rank"]), skel_off=_i64(d["skel_off"]), skel=_i64(d["skel"]),
        coeff_off=_i64(d["coeff_off"]), coeff=_f64(d["coeff"]), h=float(d["h"]))


def from_compressed_kernel(ck) -> Problem:
    spec = ck.spec
    if getattr(spec, "family", "gaussian") != "gaussian":
        raise InvalidArgumentError(f"the B200 path implements the gaussian kernel only, got {spec.family!r}")
    tree = ck.tree
    nodes = tree.nodes
    nn = len(nodes)
    rank = np.zeros(nn, np.int64)
    skel, coeff = [], []
    skel_off = np.zeros(nn + 1, np.int64)
    coeff_off = np.zeros(nn + 1, np.int64)
    for v in range(nn):
        sk = ck.skeletons[v]
        if sk is not None:
            rank[v] = sk.skel.size
            skel.append(np.asarray(sk.skel, np.int64))
            coeff.append(np.asarray(sk.coeff, np.float64).ravel())
        skel_off[v + 1] = skel_off[v] + rank[v]
        coeff_off[v + 1] = coeff_off[v] + (coeff[-1].size if sk is not None else 0)
    return Problem(
        coords=_f64(ck.points.coords), perm=_i64(tree.perm),
        node_begin=_i64([nd.begin for nd in nodes]), node_end=_i64([nd.end for nd in nodes]),
        node_left=_i64([nd.children[0] if nd.children else -1 for nd in nodes]),
        node_right=_i64([nd.children[1] if nd.children else -1 for nd in nodes]),
        rank=rank, skel_off=skel_off, skel=np.concatenate(skel) if skel else np.zeros(0, np.int64),
        coeff_off=coeff_off, coeff=np.concatenate(coeff) if coeff else np.zeros(0),
        h=float(spec.bandwidth))


def as_problem(ck) -> Problem:
    if isinstance(ck, Problem):
        return ck
    if isinstance(ck, dict):
        return from_arrays(ck)
    return from_compressed_kernel(ck)
