"""Persistence.

* Points: the reference's "f64-binary" format, restated byte for byte
  (points.py:22-24, 65-129): a 16-byte little-endian `<QQ` header (n, d)
  followed by the row-major float64 coordinates; the same validation and
  DataFormatError messages on load.
* Operator inputs (tree, skeleton ids, interpolation matrices, h) and
  factors: the KSINVASK container written by libinvaskit
  (ks_save_problem / ks_load_problem / ks_save_factor / ks_load_factor,
  include/invaskit.h; layout in csrc/container.h). A factor file carries the
  fingerprint of its operator and is refused for any other one.
"""

from __future__ import annotations

import ctypes as C
import os
import struct

import numpy as np

from . import _lib
from ._lib import KsProblem
from .errors import DataFormatError, InvalidArgumentError
from .problem import Problem, as_problem
from .solver import GpuHierFactor, _default_device, _raise

_BINARY_HEADER = struct.Struct("<QQ")  # points.py:24


def save_points(coords, path) -> None:
    """Write points in the reference's f64-binary format (points.py:82-85)."""
    x = np.ascontiguousarray(getattr(coords, "coords", coords), dtype="<f8")
    if x.ndim != 2:
        raise InvalidArgumentError(f"points must be an (n, d) array, got shape {x.shape}")
    with open(path, "wb") as fh:
        fh.write(_BINARY_HEADER.pack(x.shape[0], x.shape[1]))
        fh.write(x.tobytes())


def load_points(path) -> np.ndarray:
    """Read an f64-binary point file (points.py:107-129); (n, d) float64."""
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) < _BINARY_HEADER.size:
        raise DataFormatError(f"{path}: truncated header, {len(raw)} bytes < {_BINARY_HEADER.size}")
    n, d = _BINARY_HEADER.unpack_from(raw, 0)
    expected = _BINARY_HEADER.size + 8 * n * d
    if len(raw) != expected:
        raise DataFormatError(
            f"{path}: expected {expected} bytes for n={n}, d={d}, "
            f"got {len(raw)} (mismatch at byte offset {min(len(raw), expected)})")
    if n < 1 or d < 1:
        raise DataFormatError(f"{path}: invalid header n={n}, d={d}")
    coords = np.frombuffer(raw, dtype="<f8", offset=_BINARY_HEADER.size).reshape(n, d)
    if not np.all(np.isfinite(coords)):
        bad = int(np.flatnonzero(~np.isfinite(coords).ravel())[0])
        raise DataFormatError(f"{path}: non-finite value at byte offset {_BINARY_HEADER.size + 8 * bad}")
    return coords.astype(np.float64, copy=True)


def save_operator(source, path) -> None:
    """Write the operator inputs of `source` (a CompressedKernel, Problem or
    the plain-array dict) to `path`."""
    prob = as_problem(source)
    cp = prob.to_c()
    rc = _lib.load().ks_save_problem(C.byref(cp), os.fsencode(path))
    if rc:
        _raise(rc)


def load_operator(path) -> Problem:
    """Read operator inputs written by save_operator into a Problem."""
    lib = _lib.load()
    cp = KsProblem()
    owner = C.c_void_p()
    rc = lib.ks_load_problem(os.fsencode(path), C.byref(cp), C.byref(owner))
    if rc:
        _raise(rc)
    try:
        n, d, nn = int(cp.n), int(cp.d), int(cp.n_nodes)

        def i64(ptr, cnt):
            return np.ctypeslib.as_array(ptr, shape=(cnt,)).copy() if cnt else np.zeros(0, np.int64)

        def f64(ptr, cnt):
            return np.ctypeslib.as_array(ptr, shape=(cnt,)).copy() if cnt else np.zeros(0)

        skel_off = i64(cp.skel_off, nn + 1)
        coeff_off = i64(cp.coeff_off, nn + 1)
        return Problem(coords=f64(cp.coords, n * d).reshape(n, d), perm=i64(cp.perm, n),
                       node_begin=i64(cp.node_begin, nn), node_end=i64(cp.node_end, nn),
                       node_left=i64(cp.node_left, nn), node_right=i64(cp.node_right, nn),
                       rank=i64(cp.rank, nn), skel_off=skel_off, skel=i64(cp.skel, int(skel_off[-1])),
                       coeff_off=coeff_off, coeff=f64(cp.coeff, int(coeff_off[-1])), h=float(cp.bandwidth))
    finally:
        lib.ks_free_problem(owner)


def save_factor(hf: GpuHierFactor, path) -> None:
    """Write a factorized handle (factor buffers, lam, diagnostics) keyed to its operator."""
    cp = hf.problem.to_c()
    rc = _lib.load().ks_save_factor(hf.handle, C.byref(cp), os.fsencode(path))
    if rc:
        _raise(rc, hf.handle)


def load_factor(path, source, *, device: int | None = None) -> GpuHierFactor:
    """Recreate a factorized handle for operator `source` from a factor file
    (no refactorization); DataFormatError / InvalidArgumentError if the file is
    corrupt or belongs to another operator."""
    prob = as_problem(source)
    cp = prob.to_c()
    dev = _default_device() if device is None else int(device)
    h = C.c_void_p()
    rc = _lib.load().ks_load_factor(os.fsencode(path), C.byref(cp), dev, C.byref(h))
    if rc:
        _raise(rc)
    lam = _factor_lam(h.value)
    return GpuHierFactor(source, prob, lam, h.value, dev)


def _factor_lam(handle) -> float:
    lam = C.c_double()
    rc = _lib.load().ks_get_lam(handle, C.byref(lam))
    if rc:
        _raise(rc, handle)
    return float(lam.value)
