import sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import numpy as np
from conftest import load_golden, rel
import paper_1602_01376_b200 as ks
for case in (sys.argv[1:] or ["single", "ragged", "cfg1", "cfg2s", "cfg3s", "cfg4s", "cfg5s"]):
    g = load_golden(case)
    t0 = time.time()
    try:
        hf = ks.factorize(g, float(g["lam"]))
    except Exception as e:
        print(case, "FACTOR ERROR", type(e).__name__, e); continue
    t1 = time.time()
    herr = 0.0
    for i, v in enumerate(g["H_nodes"]):
        H = g["H"][g["H_off"][i]:g["H_off"][i + 1]]
        herr = max(herr, rel(hf.node_h(int(v)).ravel(), H))
    lerr = rel(hf.leaf_factor(int(g["leaf0_node"])), g["leaf0_L"]) if "leaf0_L" in g else -1
    u = ks.solve_many(hf, g["b"])
    zc = hf.diagnostics["z_cond"]
    zerr = max([abs(zc[int(v)] / c - 1) for v, c in zip(g["z_cond_nodes"], g["z_cond"])] or [0])
    print(f"{case}: u_err={rel(u, g['u']):.2e} H_err={herr:.2e} L_err={lerr:.2e} zcond_relerr={zerr:.2e} "
          f"t_factor+create={t1-t0:.3f}s fallback={hf.diagnostics['fallback_nodes']}", flush=True)
    hf.close()
