"""Kernel ridge regression front ends on the B200 path (solver.py:240-301).

`krr_fit` composes tree + compression + `factorize` + `solve` with the tree
permutation hidden from the caller (labels and weights in original point
order, solver.py:240-270). `krr_predict` is the dense, exact cross-kernel
matvec sum_i k(x_test_j, x_train_i) w_i (solver.py:273-301), computed by
`ks_kernel_matvec`: a DMMA Gram GEMM with the Gaussian kernel, the weights
and the row reduction fused into its epilogue, partial sums per 64-column
tile added in a fixed order (deterministic).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .errors import InvalidArgumentError
from .solver import _check_lam, _default_device, _raise, factorize, solve


def _coords(points) -> np.ndarray:
    x = getattr(points, "coords", points)
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.ndim != 2:
        raise InvalidArgumentError(f"points must be an (n, d) array, got shape {x.shape}")
    return x


def _bandwidth(spec) -> float:
    name = getattr(spec, "family", "gaussian")
    if name != "gaussian":  # the GPU path implements the Gaussian kernel (kernels.py:29-59)
        raise InvalidArgumentError(f"unsupported kernel {name!r}: the B200 path implements 'gaussian'")
    h = float(getattr(spec, "bandwidth", spec))
    if not (h > 0.0) or not np.isfinite(h):
        raise InvalidArgumentError(f"gaussian kernel needs bandwidth > 0, got {h}")
    return h


def _reference_available() -> bool:
    try:
        import kernelsolve  # noqa: F401
    except ImportError:
        return False
    return True


def krr_fit(points, spec, lam: float, y, *, leaf_size: int = 256, params=None, threads: int = 1,
            producer: str = "auto", device: int | None = None) -> np.ndarray:
    """Weights w = (K~ + lam I)^-1 y in ORIGINAL point order (solver.py:240-270).

    producer: where the operator inputs come from. "reference" runs the
    reference's build_tree + compress (the exact operator kernelsolve.krr_fit
    factors); "gpu" uses this repository's GPU producer (bit-exact tree
    restatement, GPU interpolative decomposition; same construction, not the
    same skeleton bits); "auto" prefers the reference when it is importable.
    """
    x = _coords(points)
    n = x.shape[0]
    yv = np.asarray(y, dtype=np.float64)
    if yv.ndim != 1 or yv.shape[0] != n:  # solver.py:256-259
        raise InvalidArgumentError(f"labels must be a length-{n} vector, got shape {yv.shape}")
    if not np.all(np.isfinite(yv)):  # solver.py:260-261
        raise InvalidArgumentError("labels must be finite")
    lam = _check_lam(lam)
    h = _bandwidth(spec)
    if producer == "auto":
        producer = "reference" if _reference_available() else "gpu"
    if producer == "reference":
        import kernelsolve as ref

        if params is None:
            params = ref.CompressParams()
        tree = ref.build_tree(points, leaf_size)
        source = ref.compress(points, tree, spec, params, threads=threads)
        perm = np.asarray(tree.perm, dtype=np.int64)
    elif producer == "gpu":
        from producer import make_operator_from_points

        kw = {}
        if params is not None:
            kw = {"max_rank": int(params.max_rank), "tol": float(params.tol),
                  "n_neighbors": int(params.n_neighbors), "seed": int(params.seed)}
        from .problem import from_arrays

        op = make_operator_from_points(x, leaf_size, h, **kw)
        source = from_arrays(op)
        perm = op["perm"]
    else:
        raise InvalidArgumentError(f"unknown producer {producer!r}")
    hf = factorize(source, lam, threads, device=device)
    try:
        w_perm = solve(hf, yv[perm])
    finally:
        hf.close()
    w = np.empty_like(w_perm)
    w[perm] = w_perm
    return w


def krr_predict(points_train, w, spec, points_test, *, device: int | None = None) -> np.ndarray:
    """sum_i k(x_test_j, x_train_i) w_i, dense and exact (solver.py:273-301)."""
    xtr = _coords(points_train)
    xte = _coords(points_test)
    wv = np.ascontiguousarray(w, dtype=np.float64)
    if wv.ndim != 1 or wv.shape[0] != xtr.shape[0]:  # solver.py:281-284
        raise InvalidArgumentError(f"weights must be a length-{xtr.shape[0]} vector, got shape {wv.shape}")
    if xte.shape[1] != xtr.shape[1]:  # solver.py:285-288
        raise InvalidArgumentError(f"dimension mismatch: train d={xtr.shape[1]}, test d={xte.shape[1]}")
    h = _bandwidth(spec)
    if xte.shape[0] == 0:  # solver.py:289-290
        return np.empty(0)
    out = np.empty(xte.shape[0], dtype=np.float64)
    lib = _lib.load()
    dev = _default_device() if device is None else int(device)
    rc = lib.ks_kernel_matvec(xte.ctypes.data, xte.shape[0], xtr.ctypes.data, xtr.shape[0], xtr.shape[1], h,
                              wv.ctypes.data, out.ctypes.data, dev, None)
    if rc:
        _raise(rc)
    return out
