"""Algorithmic work of the factor/solve path (fixed yardsticks).

FLOPs count the minimal standard formulation of what the reference computes,
with textbook kernel costs (GEMM 2mnk, SYRK n^2 k, TRSM n^2 k, Cholesky n^3/3,
LU 2n^3/3), from each node's actual sizes and ranks:

  leaf            m^2 d + m^3/3 + m^2 s + m s^2
  internal        2 s_l s_r d + 2 s_l s_r t + (2/3) t^3 + 2 t^2 s + 2 s (s_l^2 + s_r^2) + 2 s^2 t
  root            2 s_l s_r d + 2 s_l s_r t + (2/3) t^3

Solve bytes (fp64) stream the reference's factor set once per pass:

  leaf            8 (2 m^2 + 2 s m + 3 m q)
  internal        8 (s_l s_r + 2 t^2 + (s_l^2 + s_r^2) + 2 s t)     (B, Z twice, G, P twice)
  root            8 (s_l s_r + t^2)

Solve FLOPs (for q >= 16, where the solve crosses the fp64 ridge): every
stored matrix entry read is used in one FMA per right-hand side.
"""

from __future__ import annotations

import numpy as np


def _walk(prob):
    left, right = prob["node_left"], prob["node_right"]
    begin, end, rank = prob["node_begin"], prob["node_end"], prob["rank"]
    d = prob["coords"].shape[1]
    for v in range(len(begin)):
        if left[v] < 0:
            yield ("leaf", int(end[v] - begin[v]), int(rank[v]), 0, 0, d, v == 0)
        else:
            yield ("node", 0, int(rank[v]), int(rank[left[v]]), int(rank[right[v]]), d, v == 0)


def factor_flops(prob) -> float:
    total = 0.0
    for kind, m, s, sl, sr, d, root in _walk(prob):
        if kind == "leaf":
            total += m * m * d + m ** 3 / 3.0 + (m * m * s + m * s * s if not root else 0.0)
        else:
            t = sl + sr
            total += 2.0 * sl * sr * d + 2.0 * sl * sr * t + 2.0 / 3.0 * t ** 3
            if not root:
                total += 2.0 * t * t * s + 2.0 * s * (sl * sl + sr * sr) + 2.0 * s * s * t
    return total


def solve_bytes(prob, q: int) -> float:
    total = 0.0
    for kind, m, s, sl, sr, d, root in _walk(prob):
        if kind == "leaf":
            total += 8.0 * (2 * m * m + 2 * s * m + 3 * m * q)
        else:
            t = sl + sr
            total += 8.0 * (sl * sr + t * t) if root else 8.0 * (sl * sr + 2 * t * t + sl * sl + sr * sr + 2 * s * t)
    return total


def solve_flops(prob, q: int) -> float:
    return 2.0 * q * (solve_bytes(prob, 0) / 8.0)


def summary(prob, q: int) -> dict:
    return {"factor_flops": factor_flops(prob), "solve_bytes": solve_bytes(prob, q),
            "solve_flops": solve_flops(prob, q)}


def leaf_count(prob) -> int:
    return int(np.sum(np.asarray(prob["node_left"]) < 0))
