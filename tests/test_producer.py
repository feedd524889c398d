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
