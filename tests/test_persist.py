"""Persistence: the reference's f64-binary points
format (byte-compatible with a file the reference wrote), the operator-input
container (host-only library calls, runs on CPU) and factor files (GPU)."""
import os

import numpy as np
import pytest

import paper_1602_01376_b200 as ks
from conftest import GOLDEN


def test_points_read_reference_file_and_write_same_bytes(tmp_path):
    ref = os.path.join(GOLDEN, "points_ref.f64")
    x = ks.load_points(ref)
    assert np.array_equal(x, np.load(os.path.join(GOLDEN, "points_ref_coords.npy")))
    out = tmp_path / "p.f64"
    ks.save_points(x, out)
    assert out.read_bytes() == open(ref, "rb").read()


def test_points_format_errors(tmp_path):
    p = tmp_path / "bad.f64"
    p.write_bytes(b"\x01\x02")
    with pytest.raises(ks.DataFormatError, match="truncated header"):
        ks.load_points(p)
    x = np.arange(12, dtype=np.float64).reshape(4, 3)
    ks.save_points(x, p)
    p.write_bytes(p.read_bytes()[:-3])
    with pytest.raises(ks.DataFormatError, match="expected 112 bytes"):
        ks.load_points(p)
    x[2, 1] = np.inf
    ks.save_points(x, p)
    with pytest.raises(ks.DataFormatError, match="non-finite value at byte offset 72"):
        ks.load_points(p)


@pytest.mark.parametrize("case", ["cfg1", "ragged"])
def test_operator_round_trip_bit_exact(golden, tmp_path, case):
    g = golden(case)
    prob = ks.from_arrays(g)
    path = tmp_path / f"{case}.ksop"
    ks.save_operator(prob, path)
    back = ks.load_operator(path)
    for k in ("coords", "perm", "node_begin", "node_end", "node_left", "node_right", "rank", "skel_off", "skel",
              "coeff_off", "coeff"):
        a, b = getattr(prob, k), getattr(back, k)
        assert a.dtype == b.dtype and np.array_equal(a, b), k
    assert back.h == prob.h
    assert back.int_hash() == str(g["int_hash"])


def test_operator_file_corruption_detected(golden, tmp_path):
    prob = ks.from_arrays(golden("ragged"))
    path = tmp_path / "op.ksop"
    ks.save_operator(prob, path)
    raw = bytearray(path.read_bytes())
    # flip the lowest mantissa bit of one coordinate: still a valid file, wrong content
    at = bytes(raw).find(prob.coords.tobytes()[:64])
    assert at > 0
    raw[at + 8 * 17] ^= 0x01
    (tmp_path / "flip.ksop").write_bytes(bytes(raw))
    with pytest.raises(ks.DataFormatError, match="fingerprint"):
        ks.load_operator(tmp_path / "flip.ksop")
    (tmp_path / "short.ksop").write_bytes(bytes(raw[: len(raw) // 2]))
    with pytest.raises(ks.DataFormatError):
        ks.load_operator(tmp_path / "short.ksop")
    (tmp_path / "magic.ksop").write_bytes(b"NOTKSINV" + bytes(raw[8:]))
    with pytest.raises(ks.DataFormatError, match="not a KSINVASK"):
        ks.load_operator(tmp_path / "magic.ksop")
    with pytest.raises(ks.DataFormatError, match="cannot open"):
        ks.load_operator(tmp_path / "missing.ksop")


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["cfg1", "ragged"])
def test_factor_save_load_solves_identically(golden, tmp_path, case):
    g = golden(case)
    prob = ks.from_arrays(g)
    hf = ks.factorize(prob, float(g["lam"]))
    u = ks.solve_many(hf, g["b"])
    path = tmp_path / "f.ksfac"
    ks.save_factor(hf, path)
    diag = hf.diagnostics
    hf.close()
    hf2 = ks.load_factor(path, prob)
    assert hf2.lam == float(g["lam"])
    assert np.array_equal(ks.solve_many(hf2, g["b"]), u)
    d2 = hf2.diagnostics
    assert d2["z_cond"] == diag["z_cond"] and d2["fallback_nodes"] == diag["fallback_nodes"]
    # the handle is a normal factor: refactorize with another lam works
    hf2.refactorize(2.0 * float(g["lam"]))
    assert np.all(np.isfinite(ks.solve_many(hf2, g["b"])))
    hf2.close()


@pytest.mark.gpu
def test_factor_file_refused_for_other_operator(golden, tmp_path):
    g = golden("cfg1")
    hf = ks.factorize(ks.from_arrays(g), float(g["lam"]))
    ks.save_factor(hf, tmp_path / "f.ksfac")
    hf.close()
    with pytest.raises(ks.InvalidArgumentError, match="different operator"):
        ks.load_factor(tmp_path / "f.ksfac", ks.from_arrays(golden("ragged")))


@pytest.mark.gpu
def test_factor_save_load_with_lu_fallback_leaves(golden, tmp_path, monkeypatch):
    monkeypatch.setenv("KS_FORCE_LEAF_LU", "1")  # every leaf takes the LU path
    g = golden("cfg1")
    prob = ks.from_arrays(g)
    hf = ks.factorize(prob, float(g["lam"]))
    assert hf.diagnostics["cholesky_fallbacks"] >= 1
    u = ks.solve_many(hf, g["b"])
    fb_nodes = hf.diagnostics["fallback_nodes"]
    ks.save_factor(hf, tmp_path / "fb.ksfac")
    hf.close()
    monkeypatch.delenv("KS_FORCE_LEAF_LU")
    hf2 = ks.load_factor(tmp_path / "fb.ksfac", prob)
    assert np.array_equal(ks.solve_many(hf2, g["b"]), u)
    assert hf2.diagnostics["fallback_nodes"] == fb_nodes
    hf2.close()
