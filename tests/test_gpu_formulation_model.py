"""The augmented-factorization algebra the CUDA path uses (oracle/gpu_model.py)
reproduces the reference's reduced matrices and solution (CPU, no GPU)."""
import pytest

from conftest import rel
from oracle import gpu_model as GM
from oracle import ks_oracle as O


@pytest.mark.parametrize("case", ["cfg1", "cfg2s", "ragged", "single", "cfg5s", "cfg4s"])
def test_model_matches_reference(golden, case):
    g = golden(case)
    prob = O.Problem(g)
    F = GM.factorize_model(prob, float(g["lam"]))
    for i, v in enumerate(g["H_nodes"]):
        H = g["H"][g["H_off"][i]:g["H_off"][i + 1]]
        assert rel(F["H"][int(v)].ravel(), H) <= 1e-11, v
    u = GM.solve_model(prob, F, g["b"])
    assert rel(u, g["u"]) <= 1e-11, rel(u, g["u"])
