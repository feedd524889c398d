"""Deep-tree fixtures through the REFERENCE itself: a BASELINE configuration's
recipe at a size whose tree has 7+ levels, run through kernelsolve.build_tree +
compress (tree.py:84-172, compress.py:145-287), factorize (solver.py:92-189)
and solve_many (solver.py:200-237). Run in the build container (needs
/root/reference):

    python tests/golden/make_deep_golden.py cfg2_full   # config 2 at its BASELINE size, N = 65536
    python tests/golden/make_deep_golden.py cfg3_128k   # config 3's recipe and shape, N = 131072
    python tests/golden/make_deep_golden.py cfg4_64k    # config 4's recipe and shape, N = 65536, q = 16
    python tests/golden/make_deep_golden.py cfg5_32k    # config 5's recipe and shape (d = 784, m = 2048, s = 512), N = 32768

A fixture (tests/golden/<case>.npz) keeps what the GPU test needs and nothing
the recipe can regenerate: the integer side of the operator (tree permutation
digest, ranks, skeleton ids), per-node norms of P, the reference's solution u
for the recipe's right-hand side, its z_cond estimates, the H of levels 1-2
and the compressed-operator residual. The points and b come bit-exactly from
paper_1602_01376_b200.configs (checked against the stored digests); P is
rebuilt on the box by producer/ (bit-exact skeleton ids, P to rounding) and
compared with the stored per-node norms.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from dataclasses import asdict

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import kernelsolve as ks  # noqa: E402  (reference, build container only)

from make_golden import _cfg, build, marshal  # noqa: E402

DEEP = {
    "cfg2_full": (_cfg("cfg2", name="cfg2_full"), 1),
    "cfg3_128k": (_cfg("cfg3", name="cfg3_128k", n=131072), 2),
    "cfg4_64k": (_cfg("cfg4", name="cfg4_64k", n=65536), 16),
    "cfg5_32k": (_cfg("cfg5", name="cfg5_32k", n=32768), 1),
}


def _sha(a, dt):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=dt).tobytes()).hexdigest()


def make(case: str) -> None:
    cfg, q = DEEP[case]
    t0 = time.perf_counter()
    ck, b, t_comp = build(cfg, q)
    print(f"{case}: compress {t_comp:.1f}s", flush=True)
    a = marshal(ck)
    out = {k: a[k] for k in ("rank", "skel_off", "skel")}
    out["gen_cfg"] = np.array(json.dumps(asdict(cfg)))
    out["q"] = np.int64(q)
    out["coords_sha256"] = np.array(_sha(a["coords"], "<f8"))
    out["perm_sha256"] = np.array(_sha(a["perm"], "<i8"))
    out["b_sha256"] = np.array(_sha(b, "<f8"))
    nn = a["rank"].size
    out["coeff_norm"] = np.array([np.linalg.norm(a["coeff"][a["coeff_off"][v]:a["coeff_off"][v + 1]])
                                  for v in range(nn)])
    t1 = time.perf_counter()
    hf = ks.factorize(ck, cfg.lam, threads=os.cpu_count() or 1)
    t_fac = time.perf_counter() - t1
    print(f"{case}: factorize {t_fac:.1f}s", flush=True)
    t1 = time.perf_counter()
    u = ks.solve_many(hf, b)
    t_sol = time.perf_counter() - t1
    out["u"] = u
    dg = hf.diagnostics
    zc = sorted(dg["z_cond"].items())
    out["z_cond_nodes"] = np.array([k for k, _ in zc], np.int64)
    out["z_cond"] = np.array([v for _, v in zc], np.float64)
    out["fallback_nodes"] = np.array(dg["fallback_nodes"], np.int64)
    out["n_warnings"] = np.int64(len(dg["warnings"]))
    hs, h_off, h_nodes = [], [0], []
    for v in range(1, 7):  # levels 1 and 2: the reduced matrices everything below feeds
        if v not in hf.node_factors:
            continue
        H = hf.node_factors[v].H
        h_nodes.append(v)
        hs.append(H.ravel())
        h_off.append(h_off[-1] + H.size)
    out["H_nodes"] = np.array(h_nodes, np.int64)
    out["H_off"] = np.array(h_off, np.int64)
    out["H"] = np.concatenate(hs)
    resid = ks.hss_matvec(ck, u) + cfg.lam * u - b
    out["roundtrip"] = np.float64(np.linalg.norm(resid) / np.linalg.norm(b))
    np.savez_compressed(os.path.join(HERE, f"{case}.npz"), **out)
    print(f"{case} N={cfg.n}: {nn} nodes, ranks {sorted(set(a['rank'].tolist()))[:6]}, max z_cond "
          f"{out['z_cond'].max():.3g}, roundtrip {out['roundtrip']:.2e}, compress {t_comp:.1f}s, factor "
          f"{t_fac:.1f}s, solve {t_sol:.1f}s, total {time.perf_counter() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    for c in sys.argv[1:] or list(DEEP):
        make(c)
