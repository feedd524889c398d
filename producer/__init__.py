"""Operator-input production for benchmarks and full-size tests.

The factor/solve hot path treats (tree, skeleton ids, P) as inputs that come
from the reference's compression stage (BASELINE.json north_star). The golden
fixtures carry the reference's own inputs at small N; at BASELINE sizes the
GPU box has no reference, so `make_operator` rebuilds them: the points from
the config recipe (paper_1602_01376_b200.configs), the tree with the
bit-exact restatement in producer.tree, and skeletons/P with the batched GPU
interpolative decomposition in producer.skeletons, rows sampled as the
reference does (kNN-guided exterior rows, producer.knn).
Not part of the product path.
"""

from __future__ import annotations

import time

import numpy as np

from paper_1602_01376_b200.configs import Config, gen_points, gen_rhs

from .tree import build_tree


def make_operator(cfg: Config, device: str = "cuda", verbose: bool = False, sampling: str = "knn") -> dict:
    from .skeletons import skeletonize

    t0 = time.perf_counter()
    coords = gen_points(cfg)
    t1 = time.perf_counter()
    tree = build_tree(coords, cfg.leaf_size)
    t2 = time.perf_counter()
    sk = skeletonize(coords, tree, cfg.h, cfg.max_rank, cfg.tol, cfg.n_neighbors, cfg.seed, device, sampling)
    t3 = time.perf_counter()
    if verbose:
        print(f"[producer] {cfg.name}: points {t1 - t0:.1f}s tree {t2 - t1:.1f}s skeletons {t3 - t2:.1f}s "
              f"ranks {sorted(set(sk['rank'].tolist()))[:4]}", flush=True)
    out = {"coords": coords, "h": np.float64(cfg.h), "lam": np.float64(cfg.lam)}
    out.update(tree)
    out.update(sk)
    return out


def make_operator_from_points(coords: np.ndarray, leaf_size: int, h: float, max_rank: int = 256, tol: float = 1e-5,
                              n_neighbors: int = 32, seed: int = 0, device: str = "cuda",
                              sampling: str = "knn") -> dict:
    """Operator inputs for given points (krr_fit's GPU producer): the bit-exact
    tree restatement and the GPU skeletonization, CompressParams defaults
    (compress.py:41-69) unless overridden."""
    from .skeletons import skeletonize

    coords = np.ascontiguousarray(coords, dtype=np.float64)
    tree = build_tree(coords, leaf_size)
    sk = skeletonize(coords, tree, h, max_rank, tol, n_neighbors, seed, device, sampling)
    out = {"coords": coords, "h": np.float64(h)}
    out.update(tree)
    out.update(sk)
    return out


def make_rhs(cfg: Config, perm: np.ndarray, q: int) -> np.ndarray:
    """(n, q) right-hand side in TREE order (cli.py:270-272 convention)."""
    return gen_rhs(cfg, q).reshape(cfg.n, q)[perm]
