"""The operator producer's tree is the reference tree bit for bit (perm and
node table of the golden fixtures, which the reference built)."""
import numpy as np
import pytest

from paper_1602_01376_b200.configs import CONFIGS
from producer.tree import build_tree


@pytest.mark.parametrize("case,leaf", [("cfg1", 128), ("ragged", 100), ("single", 128), ("cfg2s", 512),
                                       ("cfg3s", 1024), ("cfg4s", 512), ("cfg5s", 256)])
def test_tree_bit_exact(golden, case, leaf):
    g = golden(case)
    t = build_tree(g["coords"], leaf)
    for k in ("perm", "node_begin", "node_end", "node_level", "node_left", "node_right"):
        assert np.array_equal(t[k], g[k]), k


@pytest.mark.parametrize("case", ["cfg1", "cfg2s", "cfg3s", "cfg4s", "cfg5s"])
def test_config_points_match_fixture(golden, case):
    from dataclasses import replace
    from paper_1602_01376_b200.configs import gen_points
    g = golden(case)
    base = CONFIGS[case.rstrip("s")]
    n, d = g["coords"].shape
    cfg = replace(base, n=n)
    assert cfg.d == d
    assert np.array_equal(gen_points(cfg), g["coords"])


def _skeletons_match(g, sk, nn):
    bad = [v for v in range(nn) if not np.array_equal(sk["skel"][sk["skel_off"][v]:sk["skel_off"][v + 1]],
                                                      g["skel"][g["skel_off"][v]:g["skel_off"][v + 1]])]
    return np.array_equal(sk["rank"], g["rank"]), bad


@pytest.mark.parametrize("case,base", [("cfg1", "cfg1"), ("cfg2s", "cfg2"), ("cfg3s", "cfg3"), ("cfg4s", "cfg4"),
                                       ("cfg5s", "cfg5"), ("ragged", "cfg1")])
def test_skeletons_bit_exact(golden, case, base):
    """The producer's skeleton ids and ranks are the reference's (the fill-up
    draw is the reference's own generator(seed, 0x726F77, node), compress.py:190;
    kNN ties toward the smaller id, tree.py:157-171), on the CPU."""
    from producer.skeletons import skeletonize
    g = golden(case)
    leaf = int((g["node_end"] - g["node_begin"])[g["node_left"] < 0].max())
    t = build_tree(g["coords"], leaf)
    sk = skeletonize(g["coords"], t, float(g["h"]), int(g["rank"].max()), CONFIGS[base].tol, 32, 0, "cpu", "knn")
    rank_ok, bad = _skeletons_match(g, sk, g["rank"].size)
    assert rank_ok and not bad, bad
    assert np.linalg.norm(sk["coeff"] - g["coeff"]) <= 1e-12 * np.linalg.norm(g["coeff"])


def _check_16k(device):
    from dataclasses import replace

    from conftest import load_golden
    from paper_1602_01376_b200.configs import gen_points
    from producer.skeletons import skeletonize
    g = load_golden("producer16k")
    cfg = replace(CONFIGS["cfg3"], n=int(g["n"]))
    x = gen_points(cfg)
    t = build_tree(x, cfg.leaf_size)
    assert np.array_equal(t["perm"], g["perm"])
    sk = skeletonize(x, t, cfg.h, cfg.max_rank, cfg.tol, cfg.n_neighbors, cfg.seed, device, "knn")
    rank_ok, bad = _skeletons_match(g, sk, g["rank"].size)
    assert rank_ok and not bad, bad
    assert abs(np.linalg.norm(sk["coeff"]) / float(g["coeff_norm"]) - 1) <= 1e-12


@pytest.mark.slow
def test_skeletons_bit_exact_16k_cpu():
    """Config 3's recipe at N = 16384 against the reference's own compression
    (tests/golden/make_producer_golden.py): identical tree, ranks and skeleton ids."""
    _check_16k("cpu")


@pytest.mark.gpu
def test_skeletons_bit_exact_16k_gpu():
    _check_16k("cuda")
