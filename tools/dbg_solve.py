import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import ctypes as C
import numpy as np
from conftest import load_golden, rel
import paper_1602_01376_b200 as ks
from paper_1602_01376_b200 import _lib
from oracle import ks_oracle as O, gpu_model as GM
case = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
g = load_golden(case)
prob = O.Problem(g)
F = GM.factorize_model(prob, float(g["lam"]))
hf = ks.factorize(g, float(g["lam"]))
u = ks.solve_many(hf, g["b"])
lib = _lib.load()
lay = np.zeros(8, np.int64); lib.ks_debug_layout(hf.handle, lay.ctypes.data_as(C.POINTER(C.c_int64)))
M, S, TP, T, R, q, nint, nl = [int(x) for x in lay]
print("layout", lay)
def dev(which, idx, count):
    out = np.zeros(count); lib.ks_debug_copy(hf.handle, which, idx, out.ctypes.data_as(C.POINTER(C.c_double)), count); return out
# model intermediates
B = g["b"]
leaves = [v for v in range(prob.n_nodes) if prob.is_leaf(v)]
for li, v in enumerate(leaves[:3]):
    L, L21 = F["leaf"][v]
    z = np.linalg.solve(L, B[prob.begin[v]:prob.end[v]])
    zd = dev(0, li, M * q).reshape(M, q)[:L.shape[0]]
    cd = dev(1, v, S * q).reshape(S, q)[:L21.shape[0]]
    print("leaf", v, "z err", rel(zd, z), "c err", rel(cd, L21 @ z))
ints = [v for lv in prob.levels_bottom_up() for v in lv if not prob.is_leaf(v)]
print("u err", rel(u, g["u"]))
# internal nodes: model y / c vs device (padded layout)
c_m, y_m = {}, {}
for v in leaves:
    L, L21 = F["leaf"][v]
    c_m[v] = L21 @ np.linalg.solve(L, B[prob.begin[v]:prob.end[v]])
for k, v in enumerate(ints):
    LU, piv, Bc, t, s_l = F["node"][v]
    l, r = int(prob.left[v]), int(prob.right[v])
    cc = np.concatenate([c_m[l], c_m[r]])
    w = np.concatenate([Bc @ c_m[r], Bc.T @ c_m[l]])
    Lu = np.tril(LU[:t, :t], -1) + np.eye(t)
    y = np.linalg.solve(Lu, GM._apply_piv(piv, w))
    y_m[v] = y
    if LU.shape[0] > t:
        c_m[v] = prob.coeff(v) @ cc + LU[t:, :t] @ y
    yd = dev(3, k, TP * q).reshape(TP, q)
    s_r = t - s_l
    yd_c = np.concatenate([yd[:s_l], yd[S:S + s_r]])
    cd = dev(1, v, S * q).reshape(S, q)[:int(prob.rank[v])] if v != 0 else None
    print("node", v, "y err", rel(yd_c, y), "c err", rel(cd, c_m[v]) if cd is not None else "-")
    if k > 40: break
