"""GPU factor/solve against the REFERENCE ITSELF on deep trees (7 levels of
internal nodes), made by tests/golden/make_deep_golden.py running
kernelsolve.compress / factorize / solve_many here:

* cfg2_full — config 2 at its BASELINE size (N = 65536, d = 18, m = 512,
  s <= 128 with the reference's variable ranks);
* cfg4_64k  — config 4's recipe and shape (d = 54, m = 512, s = 256, q = 16) at N = 65536;
* cfg3_128k — config 3's recipe and shape (d = 28, m = 1024, s = 256) at N = 131072.

The fixtures hold the reference's integer outputs and solution only; the box
rebuilds the operator with producer/ and the test first proves that operator
IS the reference's (points, permutation and right-hand side by digest, ranks and
skeleton ids element for element, P by per-node norm), then compares u
(north_star: <= 1e-10), the top reduced matrices H and the Z condition
estimates (solver.py:150, linalg.py:282-304) with the reference's.
"""
import hashlib
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, rel

pytestmark = pytest.mark.gpu


def _sha(a, dt):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=dt).tobytes()).hexdigest()


@pytest.mark.parametrize("case,pipe_min", [("cfg2_full", None), ("cfg4_64k", None), ("cfg3_128k", None),
                                           ("cfg5_32k", None), ("cfg4_64k", "1"), ("cfg3_128k", "1")])
def test_deep_tree_matches_reference(case, pipe_min, monkeypatch):
    """pipe_min = "1" (KS_PIPE_MIN=1): every subtree-local level is
    pipelined per subtree on its own stream (8-, 4-, 2- and 1-node sub-batches,
    per-level condition estimates beside the next level) in the first
    factorization and in the replayed graph of the second; each node's LU variant
    follows the replay schedule's batch size, so the two give the same bits."""
    import json

    import paper_1602_01376_b200 as ks
    from paper_1602_01376_b200.configs import Config
    from producer import make_operator, make_rhs

    if not os.path.exists(os.path.join(GOLDEN, f"{case}.npz")):
        pytest.skip(f"{case}.npz not generated")
    g = load_golden(case)  # regenerates the points and checks their digest
    kw = json.loads(str(g["gen_cfg"]))
    kw["q"] = tuple(kw["q"])
    cfg = Config(**kw)
    q = int(g["q"])
    op = make_operator(cfg)
    # the operator is the reference's: integers bit for bit, P to rounding
    assert _sha(op["coords"], "<f8") == str(g["coords_sha256"])
    assert _sha(op["perm"], "<i8") == str(g["perm_sha256"])
    assert np.array_equal(op["rank"], g["rank"])
    assert np.array_equal(op["skel_off"], g["skel_off"])
    assert np.array_equal(op["skel"], g["skel"])
    nn = op["rank"].size
    pn = np.array([np.linalg.norm(op["coeff"][op["coeff_off"][v]:op["coeff_off"][v + 1]]) for v in range(nn)])
    ok = g["coeff_norm"] > 0
    assert np.max(np.abs(pn[ok] / g["coeff_norm"][ok] - 1)) <= 1e-11
    b = make_rhs(cfg, op["perm"], q)
    assert _sha(b, "<f8") == str(g["b_sha256"])

    if pipe_min:
        monkeypatch.setenv("KS_PIPE_MIN", pipe_min)
    hf = ks.factorize(op, cfg.lam)
    if pipe_min:
        monkeypatch.delenv("KS_PIPE_MIN")
    u = ks.solve_many(hf, b)
    if pipe_min:
        assert hf.pipelined_levels()[1] >= 3  # the deep per-subtree pipeline really ran
        hf.refactorize(cfg.lam)
        assert np.array_equal(ks.solve_many(hf, b), u)
    assert u.shape == g["u"].shape
    err = rel(u, g["u"])
    assert err <= cfg.tol_u, err
    zc = hf.diagnostics["z_cond"]
    assert sorted(zc) == g["z_cond_nodes"].tolist()
    for v, c in zip(g["z_cond_nodes"].tolist(), g["z_cond"].tolist()):
        assert abs(zc[v] / c - 1) <= 1e-6, (v, zc[v], c)
    assert hf.diagnostics["cholesky_fallbacks"] == g["fallback_nodes"].size
    assert len(hf.diagnostics["warnings"]) == int(g["n_warnings"])
    for i, v in enumerate(g["H_nodes"].tolist()):
        r = int(g["rank"][v])
        H = g["H"][g["H_off"][i]:g["H_off"][i + 1]].reshape(r, r)
        assert rel(hf.node_h(v)[:r, :r], H) <= 1e-11, v
    hf.close()
