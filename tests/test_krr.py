"""KRR front ends (solver.py:240-301): the oracle pinned to the reference's
krr_fit / krr_predict outputs (tests/golden/make_krr_golden.py), and the GPU
path through ks_kernel_matvec / factorize / solve against the same fixture."""
import numpy as np
import pytest

from conftest import rel
from oracle import ks_oracle as O


def test_oracle_krr_predict_matches_reference(golden):
    g = golden("krr")
    assert rel(O.krr_predict(g["coords"], g["w"], float(g["h"]), g["x_test"]), g["pred"]) <= 1e-14
    assert rel(O.krr_predict(g["x3"], g["w3"], 0.4, g["x3_test"]), g["pred3"]) <= 1e-14


def test_oracle_krr_weights_match_reference(golden):
    g = golden("krr")
    w = O.krr_weights(O.Problem(g), float(g["lam"]), g["y"])
    assert rel(w, g["w"]) <= 1e-11, rel(w, g["w"])


def test_krr_argument_checks_cpu():
    import paper_1602_01376_b200 as ks

    x = np.zeros((10, 3))
    with pytest.raises(ks.InvalidArgumentError):
        ks.krr_predict(x, np.zeros(9), 0.5, x)
    with pytest.raises(ks.InvalidArgumentError):
        ks.krr_predict(x, np.zeros(10), 0.5, np.zeros((4, 2)))
    with pytest.raises(ks.InvalidArgumentError):
        ks.krr_fit(x, 0.5, 1.0, np.zeros(9))
    with pytest.raises(ks.InvalidArgumentError):
        ks.krr_fit(x, 0.5, 1.0, np.full(10, np.nan))
    with pytest.raises(ks.InvalidArgumentError):
        ks.krr_fit(x, 0.5, -1.0, np.zeros(10))
    assert ks.krr_predict(x, np.zeros(10), 0.5, np.zeros((0, 3))).shape == (0,)


@pytest.mark.gpu
def test_gpu_krr_predict_matches_reference(golden):
    import paper_1602_01376_b200 as ks

    g = golden("krr")
    p = ks.krr_predict(g["coords"], g["w"], float(g["h"]), g["x_test"])
    assert rel(p, g["pred"]) <= 1e-12, rel(p, g["pred"])
    p3 = ks.krr_predict(g["x3"], g["w3"], 0.4, g["x3_test"])  # odd d, one test point
    assert rel(p3, g["pred3"]) <= 1e-12, rel(p3, g["pred3"])


@pytest.mark.gpu
def test_gpu_krr_predict_large_blocks_deterministic():
    import paper_1602_01376_b200 as ks

    rng = np.random.default_rng(5)
    xtr, xte = rng.random((20000, 7)), rng.random((3000, 7))
    w = rng.standard_normal(20000)
    p1 = ks.krr_predict(xtr, w, 0.7, xte)
    p2 = ks.krr_predict(xtr, w, 0.7, xte)
    assert np.array_equal(p1, p2)
    sel = rng.choice(3000, 64, replace=False)
    ref = O.krr_predict(xtr, w, 0.7, xte[sel])
    assert rel(p1[sel], ref) <= 1e-12, rel(p1[sel], ref)


@pytest.mark.gpu
def test_gpu_krr_fit_composition_matches_reference(golden):
    """krr_fit's tree-order solve and perm scatter on the reference's own operator."""
    import paper_1602_01376_b200 as ks

    g = golden("krr")
    hf = ks.factorize(ks.from_arrays(g), float(g["lam"]))
    perm = g["perm"]
    w_perm = ks.solve(hf, g["y"][perm])
    w = np.empty_like(w_perm)
    w[perm] = w_perm
    assert rel(w, g["w"]) <= 1e-10, rel(w, g["w"])


@pytest.mark.gpu
def test_gpu_krr_fit_gpu_producer_end_to_end(golden):
    """krr_fit with the GPU producer: same construction (tree bit-exact,
    GPU skeletons), so the weights agree with the reference's up to the
    compression tolerance, and predictions on the training points match."""
    import paper_1602_01376_b200 as ks

    g = golden("krr")

    class Params:
        max_rank, tol, n_neighbors, seed = int(g["max_rank"]), 1e-5, 32, 0

    w = ks.krr_fit(g["coords"], float(g["h"]), float(g["lam"]), g["y"], leaf_size=int(g["leaf_size"]),
                   params=Params, producer="gpu")
    assert np.all(np.isfinite(w))
    assert rel(w, g["w"]) <= 1e-3, rel(w, g["w"])
    p = ks.krr_predict(g["coords"], w, float(g["h"]), g["x_test"])
    assert rel(p, g["pred"]) <= 1e-3, rel(p, g["pred"])
