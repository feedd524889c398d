import sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
from dataclasses import replace
import paper_1602_01376_b200 as ks
from paper_1602_01376_b200.configs import CONFIGS
from producer import make_operator, make_rhs
for name, n in [("cfg2", None), ("cfg3", None)]:
    cfg = CONFIGS[name] if n is None else replace(CONFIGS[name], n=n)
    t0 = time.time()
    op = make_operator(cfg, verbose=True)
    t1 = time.time()
    hf = ks.factorize(op, cfg.lam)
    b = make_rhs(cfg, op["perm"], 1)
    u = ks.solve_many(hf, b)
    r = ks.hss_matvec(hf, u) + cfg.lam * u - b
    zc = hf.diagnostics["z_cond"]
    ranks = op["rank"]
    print(name, f"producer {t1-t0:.1f}s  ranks min/max {ranks[1:].min()}/{ranks.max()}  max z_cond {max(zc.values()):.3g}  residual {np.linalg.norm(r)/np.linalg.norm(b):.2e}", flush=True)
    hf.close()
