"""Pin the CPU oracle (oracle/ks_oracle.py) against the reference's own outputs.

The fixtures were produced by running /root/reference's kernelsolve
(tests/golden/make_golden.py); these tests run anywhere (no reference needed).
"""
import numpy as np
import pytest

from conftest import rel
from oracle import ks_oracle as O

SOLVE_CASES = ["cfg1", "cfg2s", "cfg3s", "cfg4s", "cfg5s", "cfg5m", "ragged", "single"]


@pytest.fixture(scope="module")
def factored(golden):
    cache = {}

    def get(name):
        if name not in cache:
            g = golden(name)
            prob = O.Problem(g)
            cache[name] = (g, prob, O.factorize(prob, float(g["lam"])))
        return cache[name]

    return get


@pytest.mark.parametrize("case", SOLVE_CASES)
def test_oracle_solution_matches_reference(factored, case):
    g, prob, of = factored(case)
    u = O.solve_many_telescoping(of, g["b"])
    assert rel(u, g["u"]) <= 1e-12, rel(u, g["u"])


@pytest.mark.parametrize("case", ["cfg1", "ragged", "cfg5s"])
def test_oracle_recursive_solve_matches_reference(factored, case):
    g, prob, of = factored(case)
    u = O.solve_many_recursive(of, g["b"])
    assert rel(u, g["u"]) <= 1e-13


def test_oracle_multi_rhs(factored):
    g, prob, of = factored("cfg1")
    assert rel(O.solve_many_telescoping(of, g["b3"]), g["u3"]) <= 1e-12


@pytest.mark.parametrize("case", SOLVE_CASES)
def test_oracle_reduced_matrices(factored, case):
    g, prob, of = factored(case)
    for i, v in enumerate(g["H_nodes"]):
        H = g["H"][g["H_off"][i]:g["H_off"][i + 1]]
        mine = of.reduced[int(v)].ravel()
        assert rel(mine, H) <= 1e-12, (v, rel(mine, H))


@pytest.mark.parametrize("case", SOLVE_CASES + ["illcond"])
def test_oracle_diagnostics(factored, case):
    g, prob, of = factored(case)
    zc = of.diagnostics["z_cond"]
    assert sorted(zc) == g["z_cond_nodes"].tolist()
    mine = np.array([zc[int(v)] for v in g["z_cond_nodes"]])
    if mine.size:
        assert np.allclose(mine, g["z_cond"], rtol=1e-6)
    assert of.diagnostics["fallback_nodes"] == g["fallback_nodes"].tolist()
    assert len(of.diagnostics["warnings"]) == int(g["n_warnings"])


@pytest.mark.parametrize("case,exc", [("singular", O.Singular), ("illcond_hard", O.IllConditioned),
                                      ("leaf_not_spd", O.Singular)])
def test_oracle_error_paths(golden, case, exc):
    """The oracle raises where the reference raised (tests/golden/make_error_golden.py)."""
    g = golden(case)
    with pytest.raises(exc) as ei:
        O.factorize(O.Problem(g), float(g["lam"]))
    if case == "illcond_hard":
        assert ei.value.node_id == int(g["error_node"])
        assert np.isclose(ei.value.cond_estimate, float(g["error_cond"]), rtol=1e-6)


def test_oracle_leaf_factor(factored):
    g, prob, of = factored("cfg1")
    f, fb = of.leaf[int(g["leaf0_node"])]
    assert not fb
    assert rel(f.lower, g["leaf0_L"]) <= 1e-14


def test_oracle_matvec_roundtrip(factored):
    g, prob, of = factored("cfg1")
    u = g["u"][:, 0]
    r = O.hss_matvec(prob, u) + float(g["lam"]) * u - g["b"][:, 0]
    assert np.linalg.norm(r) / np.linalg.norm(g["b"]) <= 1e-11


# ---- the LAPACK-backed fast mode (oracle/ks_fast.py), same bar ----
@pytest.mark.parametrize("case", SOLVE_CASES)
def test_fast_oracle_matches_reference(golden, case):
    from oracle import ks_fast as OF
    g = golden(case)
    ff = OF.factorize(O.Problem(g), float(g["lam"]))
    u = OF.solve_many(ff, g["b"])
    assert rel(u, g["u"]) <= 1e-12, rel(u, g["u"])
    for i, v in enumerate(g["H_nodes"]):
        H = g["H"][g["H_off"][i]:g["H_off"][i + 1]]
        assert rel(ff.reduced[int(v)].ravel(), H) <= 1e-12, (int(v), rel(ff.reduced[int(v)].ravel(), H))
    zc = OF.diagnostics(ff)["z_cond"]
    assert sorted(zc) == g["z_cond_nodes"].tolist()
    if zc:
        assert np.allclose([zc[int(v)] for v in g["z_cond_nodes"]], g["z_cond"], rtol=1e-6)


def test_fast_oracle_error_paths(golden):
    from oracle import ks_fast as OF
    g = golden("illcond_hard")
    with pytest.raises(O.IllConditioned) as ei:
        OF.factorize(O.Problem(g), float(g["lam"]))
    assert ei.value.node_id == int(g["error_node"])
    g = golden("singular")
    with pytest.raises(O.Singular):
        OF.factorize(O.Problem(g), float(g["lam"]))
