"""Generate the golden fixtures by running the REFERENCE `kernelsolve` package.

Run in the build container (needs /root/reference, which does not exist on the
GPU box):  python tests/golden/make_golden.py [case ...]

Each fixture `tests/golden/<case>.npz` holds the operator inputs exactly as the
reference compression produced them (points, tree perm and node table,
skeleton ids, interpolation matrices P) plus the reference's outputs on them:
u = kernelsolve.solve_many(factorize(ck, lam), b) (the recursive solve at
solver.py:200-237), every reduced matrix H (solver.py:135,163), the first
leaf's Cholesky factor (solver.py:126), the Z condition estimates and the
diagnostics (solver.py:175-188), and the compressed-operator residual from
kernelsolve.hss_matvec (compress.py:352-411).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np
from dataclasses import asdict

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import kernelsolve as ks  # noqa: E402  (reference, build container only)

from paper_1602_01376_b200.configs import CONFIGS, gen_points, gen_rhs, Config  # noqa: E402


def _cfg(base, **kw):
    from dataclasses import replace
    return replace(CONFIGS[base], **kw)


# name -> (config, q, lam override or None, points override or None)
CASES = {
    # config 1 at full size: the reference's own CPU-runnable case
    "cfg1": (_cfg("cfg1"), 1),
    # configs 2-5 recipes at reduced N with the full (m, s, d, h, lambda)
    "cfg2s": (_cfg("cfg2", name="cfg2s", n=4096), 1),
    "cfg3s": (_cfg("cfg3", name="cfg3s", n=4096), 2),
    "cfg4s": (_cfg("cfg4", name="cfg4s", n=2048), 16),
    "cfg5s": (_cfg("cfg5", name="cfg5s", n=1024, leaf_size=256, max_rank=64), 1),
    # config 5 at its own leaf/rank shape (m=2048, s=512, d=784, lambda=0.01):
    # 4 leaves, 2 non-root internal nodes (t = 1024) and the root
    "cfg5m": (_cfg("cfg5", name="cfg5m", n=8192), 1),
    # ragged tree: leaves on two adjacent depths, sizes 50/51/100 (tree.py:115-127)
    "ragged": (_cfg("cfg1", name="ragged", n=803, leaf_size=100, max_rank=32), 2),
    # a single leaf: the root is the whole problem (no skeletons at all)
    "single": (_cfg("cfg1", name="single", n=100, leaf_size=128, max_rank=32), 1),
    # wide bandwidth, tiny lambda: Z conditioning warnings territory
    "illcond": (_cfg("cfg1", name="illcond", n=512, d=2, h=3.0, lam=1e-9,
                     leaf_size=64, max_rank=32), 1),
}


def build(cfg: Config, q: int):
    coords = gen_points(cfg)
    if cfg.recipe == "cfg1":
        ref = ks.gen_synthetic("uniform-cube", cfg.n, cfg.d, seed=cfg.seed).coords
        assert np.array_equal(ref, coords), "uniform-cube recipe drifted from points.py"
    pts = ks.PointSet(coords)
    tree = ks.build_tree(pts, cfg.leaf_size)
    spec = ks.KernelSpec("gaussian", bandwidth=cfg.h)
    params = ks.CompressParams(tol=cfg.tol, max_rank=cfg.max_rank,
                               n_neighbors=min(cfg.n_neighbors, cfg.n - 1), seed=cfg.seed)
    t0 = time.perf_counter()
    ck = ks.compress(pts, tree, spec, params)
    t_comp = time.perf_counter() - t0
    b = gen_rhs(cfg, q).reshape(cfg.n, q)[tree.perm]
    return ck, b, t_comp


def marshal(ck) -> dict:
    tree = ck.tree
    nn = len(tree.nodes)
    out = {
        "coords": ck.points.coords,
        "perm": tree.perm.astype(np.int64),
        "node_begin": np.array([nd.begin for nd in tree.nodes], np.int64),
        "node_end": np.array([nd.end for nd in tree.nodes], np.int64),
        "node_level": np.array([nd.level for nd in tree.nodes], np.int64),
        "node_left": np.array([nd.children[0] if nd.children else -1 for nd in tree.nodes], np.int64),
        "node_right": np.array([nd.children[1] if nd.children else -1 for nd in tree.nodes], np.int64),
        "h": np.float64(ck.spec.bandwidth),
    }
    rank = np.zeros(nn, np.int64)
    skel, coeff = [], []
    skel_off, coeff_off = [0], [0]
    for v in range(nn):
        sk = ck.skeletons[v]
        if sk is not None:
            rank[v] = sk.rank
            skel.append(sk.skel.astype(np.int64))
            coeff.append(sk.coeff.ravel())
            assert sk.coeff.shape == (sk.rank, sk.cand.size)
        skel_off.append(skel_off[-1] + (sk.rank if sk is not None else 0))
        coeff_off.append(coeff_off[-1] + (sk.coeff.size if sk is not None else 0))
    out["rank"] = rank
    out["skel_off"] = np.array(skel_off, np.int64)
    out["skel"] = np.concatenate(skel) if skel else np.zeros(0, np.int64)
    out["coeff_off"] = np.array(coeff_off, np.int64)
    out["coeff"] = np.concatenate(coeff) if coeff else np.zeros(0)
    return out


def int_hash(arrs: dict) -> str:
    h = hashlib.sha256()
    for k in ("perm", "node_begin", "node_end", "node_level", "node_left", "node_right",
              "rank", "skel_off", "skel"):
        h.update(np.ascontiguousarray(arrs[k], dtype="<i8").tobytes())
    return h.hexdigest()


# fixtures too large to carry their points: the loader regenerates them from
# the recipe (bit-exact, checked against the stored sha256)
NO_COORDS = {"cfg5m"}


def make(case: str) -> None:
    cfg, q = CASES[case]
    ck, b, t_comp = build(cfg, q)
    arrs = marshal(ck)
    if case in NO_COORDS:
        c = np.ascontiguousarray(arrs.pop("coords"), dtype="<f8")
        arrs["coords_sha256"] = np.array(hashlib.sha256(c.tobytes()).hexdigest())
        arrs["gen_cfg"] = np.array(json.dumps(asdict(cfg)))
    arrs["lam"] = np.float64(cfg.lam)
    arrs["b"] = b
    arrs["int_hash"] = np.array(int_hash(arrs))
    t0 = time.perf_counter()
    try:
        hf = ks.factorize(ck, cfg.lam)
    except ks.KernelSolveError as exc:  # error cases keep the expected exception
        arrs["expect_error"] = np.array(type(exc).__name__)
        arrs["error_node"] = np.int64(getattr(exc, "node_id", -1))
        np.savez_compressed(os.path.join(HERE, f"{case}.npz"), **arrs)
        print(f"{case}: reference raised {type(exc).__name__}: {exc}")
        return
    t_fac = time.perf_counter() - t0
    t0 = time.perf_counter()
    u = ks.solve_many(hf, b)
    t_sol = time.perf_counter() - t0
    arrs["u"] = u
    if case == "cfg1":  # a multi-RHS solve on the same factor (solve_many, solver.py:200)
        b3 = np.random.default_rng(3).standard_normal((cfg.n, 3))
        arrs["b3"] = b3
        arrs["u3"] = ks.solve_many(hf, b3)
    dg = hf.diagnostics
    zc = sorted(dg["z_cond"].items())
    arrs["z_cond_nodes"] = np.array([k for k, _ in zc], np.int64)
    arrs["z_cond"] = np.array([v for _, v in zc], np.float64)
    arrs["fallback_nodes"] = np.array(dg["fallback_nodes"], np.int64)
    arrs["n_warnings"] = np.int64(len(dg["warnings"]))
    # reduced matrices H of every non-root node (leaf: solver.py:135, internal: :163)
    hs, h_off, h_nodes = [], [0], []
    for v in range(len(ck.tree.nodes)):
        if case in NO_COORDS and v in hf.leaf_factors and v != min(hf.leaf_factors):
            continue  # keep the large fixture small: internal H plus the first leaf's
        if v in hf.leaf_factors and ck.tree.nodes[v].size < ck.n:
            P = ck.skeletons[v].coeff
            H = P @ ks.dense_solve(hf.leaf_factors[v].factor, P.T)
            H = 0.5 * (H + H.T)
        elif v in hf.node_factors and hf.node_factors[v].H is not None:
            H = hf.node_factors[v].H
        else:
            continue
        h_nodes.append(v)
        hs.append(H.ravel())
        h_off.append(h_off[-1] + H.size)
    arrs["H_nodes"] = np.array(h_nodes, np.int64)
    arrs["H_off"] = np.array(h_off, np.int64)
    arrs["H"] = np.concatenate(hs) if hs else np.zeros(0)
    first_leaf = min(hf.leaf_factors)
    lf = hf.leaf_factors[first_leaf].factor
    arrs["leaf0_node"] = np.int64(first_leaf)
    if lf.size <= 512:  # keep fixtures small
        arrs["leaf0_L"] = lf.lower if lf.kind == "cholesky" else lf.lu
    resid = ks.hss_matvec(ck, u) + cfg.lam * u - b
    arrs["roundtrip"] = np.float64(np.linalg.norm(resid) / np.linalg.norm(b))
    np.savez_compressed(os.path.join(HERE, f"{case}.npz"), **arrs)
    print(f"{case}: n={cfg.n} leaves={len(hf.leaf_factors)} nodes={len(hf.node_factors)} "
          f"ranks={sorted(set(arrs['rank'].tolist()))[:6]} max_zcond={arrs['z_cond'].max() if zc else 0:.3g} "
          f"fallbacks={dg['cholesky_fallbacks']} warnings={len(dg['warnings'])} "
          f"roundtrip={arrs['roundtrip']:.2e} compress={t_comp:.1f}s factor={t_fac:.1f}s solve={t_sol:.1f}s")


if __name__ == "__main__":
    for c in sys.argv[1:] or list(CASES):
        make(c)
