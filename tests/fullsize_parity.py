"""Full-size parity at the BASELINE configurations (test infrastructure).

    python tests/fullsize_parity.py [cfg3 cfg4 ...] [--out profiles/r02_fullsize_parity.json]

For each config at its BASELINE N: the operator inputs come from the producer
(the box has no reference; SURVEY §8(d) recipes, bit-exact tree), the GPU
factorizes and solves through the public API, and the LAPACK-backed oracle
(oracle/ks_fast.py, the reference's algorithm incl. its refinement steps,
pinned to the reference's golden fixtures) factorizes and solves the SAME
operator on the host. Reported: rel L2 error of u (north_star: <= 1e-10,
1e-8 for config 5), max relative error of the reduced matrices H of the top
levels, max relative difference of the Z condition estimates, timings.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))


def run(name: str) -> dict:
    import torch

    import paper_1602_01376_b200 as ks
    from oracle import ks_fast as OF
    from oracle import ks_oracle as O
    from paper_1602_01376_b200.configs import CONFIGS
    from producer import make_operator, make_rhs

    base, _, n_override = name.partition(":")  # "cfg5:131072" = config 5's recipe and shapes at a reduced N
    cfg = CONFIGS[base]
    if n_override:
        cfg = cfg.scaled(int(n_override), suffix=f"@{n_override}")
    q = max(cfg.q)
    t0 = time.perf_counter()
    op = make_operator(cfg)
    t1 = time.perf_counter()
    b = make_rhs(cfg, op["perm"], q)
    hf = ks.factorize(op, cfg.lam)
    u = ks.solve_many(hf, b)
    zc_gpu = hf.diagnostics["z_cond"]
    prob = O.Problem(op)
    lev = prob.level
    top = [v for v in range(1, prob.n_nodes) if lev[v] <= 3]
    H_gpu = {v: hf.node_h(v) for v in top}
    hf.close()
    torch.cuda.empty_cache()
    t2 = time.perf_counter()
    ff = OF.factorize(prob, cfg.lam)
    u_ref = OF.solve_many(ff, b)
    t3 = time.perf_counter()
    err = float(np.linalg.norm(u - u_ref) / np.linalg.norm(u_ref))
    h_err = max(float(np.linalg.norm(H_gpu[v] - ff.reduced[v]) / np.linalg.norm(ff.reduced[v])) for v in top)
    zc_ref = OF.diagnostics(ff)["z_cond"]
    z_err = max(abs(zc_gpu[v] / c - 1.0) for v, c in zc_ref.items())
    return {"config": cfg.name, "n": cfg.n, "d": cfg.d, "leaf": cfg.leaf_size, "rank": cfg.max_rank, "lambda": cfg.lam,
            "q": q, "tol_u": cfg.tol_u, "u_rel_err": err, "H_top_levels_max_rel_err": h_err,
            "H_nodes_checked": len(top), "z_cond_max_rel_diff": z_err, "z_cond_max": max(zc_ref.values()),
            "producer_s": t1 - t0, "gpu_s": t2 - t1, "oracle_s": t3 - t2,
            "oracle": "oracle/ks_fast.py (LAPACK restatement of solver.py:92-237, refinement steps included)",
            "operator": "producer (config recipe points, bit-exact tree, GPU skeletonization)"}


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    out = None
    if "--out" in sys.argv:
        out = sys.argv[sys.argv.index("--out") + 1]
        args = [a for a in args if a != out]
    res = [run(c) for c in (args or ["cfg3", "cfg4"])]
    for r in res:
        print(json.dumps(r), flush=True)
    if out:
        with open(out, "w") as fh:
            json.dump(res, fh, indent=1)
