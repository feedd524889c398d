"""Small factor + solve for compute-sanitizer (one tool per run): config-1 golden
operator with every level through the persistent LU, then through the launch
sequence with 32-column panels."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import paper_1602_01376_b200 as ks
with np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "cfg1.npz")) as z:
    g = {k: z[k] for k in z.files}
for env in ({"KS_SLAB_MAX": "100000"}, {"KS_SLAB_MAX": "0", "KS_PANEL_W": "32"}):
    os.environ.update(env)
    hf = ks.factorize(g, float(g["lam"]))
    hf.refactorize(float(g["lam"]))
    u = ks.solve_many(hf, g["b"])
    print(env, "rel err", np.linalg.norm(u - g["u"]) / np.linalg.norm(g["u"]))
    hf.close()
    for k in env:
        del os.environ[k]
