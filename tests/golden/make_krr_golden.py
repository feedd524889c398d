"""Golden fixture for the KRR front ends, by running the REFERENCE package:
kernelsolve.krr_fit / krr_predict (solver.py:240-301).

Run in the build container:  python tests/golden/make_krr_golden.py
Writes tests/golden/krr.npz: training points, labels, the operator inputs the
reference's krr_fit built internally (tree + compress with the same
arguments, marshalled like the solver fixtures) so the GPU box can replay the
composition without the reference, the weights w (original order), test
points and krr_predict's output.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import kernelsolve as ks  # noqa: E402  (reference, build container only)

from make_golden import int_hash, marshal  # noqa: E402


def main() -> None:
    n, d, leaf, lam, h = 1536, 5, 96, 0.3, 0.9
    pts = ks.gen_synthetic("uniform-cube", n, d, seed=7)
    rng = np.random.default_rng(11)
    y = np.sin(3.0 * pts.coords[:, 0]) + 0.1 * rng.standard_normal(n)
    spec = ks.KernelSpec("gaussian", bandwidth=h)
    params = ks.CompressParams(max_rank=48)
    w = ks.krr_fit(pts, spec, lam, y, leaf_size=leaf, params=params)
    # the operator krr_fit factored (same deterministic tree + compress call)
    tree = ks.build_tree(pts, leaf)
    ck = ks.compress(pts, tree, spec, params)
    arrs = marshal(ck)
    arrs["int_hash"] = np.array(int_hash(arrs))
    test = ks.gen_synthetic("uniform-cube", 333, d, seed=8)
    pred = ks.krr_predict(pts, w, spec, test)
    arrs.update({"y": y, "w": w, "lam": np.float64(lam), "leaf_size": np.int64(leaf), "max_rank": np.int64(48),
                 "x_test": test.coords, "pred": pred})
    # odd dimension and a single test point through krr_predict as well
    pts3 = ks.gen_synthetic("uniform-cube", 257, 3, seed=9)
    w3 = rng.standard_normal(257)
    t3 = ks.gen_synthetic("uniform-cube", 1, 3, seed=10)
    arrs.update({"x3": pts3.coords, "w3": w3, "x3_test": t3.coords,
                 "pred3": ks.krr_predict(pts3, w3, ks.KernelSpec("gaussian", bandwidth=0.4), t3)})
    np.savez_compressed(os.path.join(HERE, "krr.npz"), **arrs)
    print(f"krr: n={n} d={d} ranks={sorted(set(arrs['rank'].tolist()))[:5]} |w|={np.linalg.norm(w):.3g}")


if __name__ == "__main__":
    main()
