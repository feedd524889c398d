"""CPU-side checks of the drop-in boundary: the C-ABI library loads and exports
every entry point include/invaskit.h declares, argument validation mirrors
the reference (solver.py:101-103, 195-212), and the marshalling of a
reference-shaped CompressedKernel is exact. No device calls."""
import os
import re
from types import SimpleNamespace

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    txt = open(os.path.join(ROOT, "include", "invaskit.h")).read()
    return sorted(set(re.findall(r"\b(ks_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_1602_01376_b200 import _lib
    lib = _lib.load()
    names = _declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)
    assert b"sm_100a" in lib.ks_version()


def test_library_exports_probe_hooks():
    """tools/ probes bind the exports declared in include/invaskit_probe.h."""
    from paper_1602_01376_b200 import _lib
    lib = _lib.load()
    txt = open(os.path.join(ROOT, "include", "invaskit_probe.h")).read()
    names = sorted(set(re.findall(r"\b(ks_[a-z0-9_]+)\s*\(", txt)))
    assert names == ["ks_probe_panel", "ks_slab_trace"]
    for n in names:
        assert hasattr(lib, n), n


def test_library_is_sm100a_only():
    import subprocess
    so = os.path.join(ROOT, "paper_1602_01376_b200", "libinvaskit.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_lambda_validation_before_any_device_work(golden):
    import paper_1602_01376_b200 as ks
    g = golden("single")
    for bad in (-1.0, float("nan"), float("inf")):
        with pytest.raises(ks.InvalidArgumentError):
            ks.factorize(g, bad)


def test_marshal_compressed_kernel_matches_arrays(golden):
    """A duck-typed reference CompressedKernel marshals to the fixture arrays."""
    from paper_1602_01376_b200.problem import from_arrays, from_compressed_kernel
    g = golden("ragged")
    nn = g["node_begin"].size
    nodes = []
    for v in range(nn):
        ch = None if g["node_left"][v] < 0 else (int(g["node_left"][v]), int(g["node_right"][v]))
        nodes.append(SimpleNamespace(begin=int(g["node_begin"][v]), end=int(g["node_end"][v]), children=ch))
    sks = []
    for v in range(nn):
        r = int(g["rank"][v])
        if r == 0:
            sks.append(None)
            continue
        sk = g["skel"][g["skel_off"][v]:g["skel_off"][v + 1]]
        cf = g["coeff"][g["coeff_off"][v]:g["coeff_off"][v + 1]].reshape(r, -1)
        sks.append(SimpleNamespace(skel=sk, coeff=cf))
    ck = SimpleNamespace(points=SimpleNamespace(coords=g["coords"]), tree=SimpleNamespace(perm=g["perm"], nodes=nodes),
                         skeletons=sks, spec=SimpleNamespace(family="gaussian", bandwidth=float(g["h"])))
    a, b = from_compressed_kernel(ck), from_arrays(g)
    for k in ("coords", "perm", "node_begin", "node_end", "node_left", "node_right", "rank", "skel_off", "skel",
              "coeff_off", "coeff"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    assert a.int_hash() == str(g["int_hash"])


def test_marshal_rejects_non_gaussian():
    import paper_1602_01376_b200 as ks
    from paper_1602_01376_b200.problem import from_compressed_kernel
    ck = SimpleNamespace(spec=SimpleNamespace(family="laplace", bandwidth=1.0))
    with pytest.raises(ks.InvalidArgumentError):
        from_compressed_kernel(ck)


def test_yardstick_matches_survey_config3_figure():
    """F = 1.178 TFLOP for config 3 on a perfect tree."""
    from paper_1602_01376_b200 import yardstick
    L, m, s, d = 1024, 1024, 256, 28
    nn = 2 * L - 1
    left = np.full(nn, -1)
    right = np.full(nn, -1)
    for v in range(L - 1):
        left[v], right[v] = 2 * v + 1, 2 * v + 2
    begin = np.zeros(nn, np.int64)
    end = np.zeros(nn, np.int64)
    for v in range(nn):
        lev = int(np.floor(np.log2(v + 1)))
        idx = v - (2 ** lev - 1)
        size = (L * m) >> lev
        begin[v], end[v] = idx * size, (idx + 1) * size
    rank = np.full(nn, s)
    rank[0] = 0
    prob = {"node_left": left, "node_right": right, "node_begin": begin, "node_end": end, "rank": rank,
            "coords": np.zeros((1, d))}
    assert abs(yardstick.factor_flops(prob) / 1e12 - 1.178) < 0.001
    assert abs(yardstick.solve_bytes(prob, 1) / 1e9 - 29.54) < 0.05
