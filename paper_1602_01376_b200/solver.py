"""Drop-in `factorize` / `solve` / `solve_many` on the B200 (sm_100a) library.

Same signatures, argument meaning, return shapes, errors and diagnostics keys
as the reference (`/root/reference/pkg/src/kernelsolve/solver.py:92-237`):

    hf = factorize(ck, lam, threads=1)   # solver.py:92
    x  = solve(hf, b)                    # solver.py:192   b: (n,) tree order
    X  = solve_many(hf, B)               # solver.py:200   B: (n, q) tree order

All arithmetic runs in libinvaskit.so on the GPU (no CPU fallback). `threads`
is accepted for signature compatibility and ignored: the output does not
depend on it (the reference's determinism contract, cli.py:488-511).
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib
from ._lib import (KS_ERR_CUDA, KS_ERR_ILL_COND, KS_ERR_INVALID, KS_ERR_IO, KS_ERR_NOT_SPD, KS_ERR_SINGULAR,
                   KS_ERR_UNSUPPORTED, KsDiag)
from .errors import (
    DataFormatError,
    DeviceError,
    IllConditionedError,
    InvalidArgumentError,
    KernelSolveError,
    NotSPDError,
    SingularMatrixError,
)
from .problem import Problem, as_problem

_COND_WARN = 1e10  # solver.py:51


def _raise(rc: int, handle=None):
    msg = _lib.last_error()
    if rc == KS_ERR_INVALID:
        raise InvalidArgumentError(msg)
    if rc == KS_ERR_NOT_SPD:
        raise NotSPDError(msg)
    if rc == KS_ERR_SINGULAR:
        raise SingularMatrixError(msg)
    if rc == KS_ERR_ILL_COND:
        d = KsDiag()
        _lib.load().ks_get_diag(handle, C.byref(d))
        raise IllConditionedError(int(d.error_node), float(d.error_cond))
    if rc in (KS_ERR_CUDA,):
        raise DeviceError(msg)
    if rc == KS_ERR_UNSUPPORTED:
        raise InvalidArgumentError(msg)
    if rc == KS_ERR_IO:
        raise DataFormatError(msg)
    raise KernelSolveError(f"libinvaskit error {rc}: {msg}")


def _default_device() -> int:
    return int(os.environ.get("LOCAL_RANK", "0"))


class GpuHierFactor:
    """Result of `factorize`: device-resident factors plus the reference's
    HierFactor surface (`ck`, `lam`, `n`, `diagnostics`, solver.py:77-89).
    Immutable after return; concurrent solves on one factor are allowed."""

    def __init__(self, ck, problem: Problem, lam: float, handle: int, device: int):
        self.ck = ck
        self.problem = problem
        self.lam = lam
        self._h = handle
        self.device = device
        self.diagnostics = self._read_diagnostics()

    @property
    def n(self) -> int:
        return self.problem.n

    @property
    def handle(self) -> int:
        if not self._h:
            raise InvalidArgumentError("factor has been released")
        return self._h

    def _read_diagnostics(self) -> dict:
        lib = _lib.load()
        nn = max(self.problem.n_nodes, 1)
        nodes = np.zeros(nn, np.int64)
        conds = np.zeros(nn, np.float64)
        cnt = lib.ks_get_z_cond(self._h, nodes.ctypes.data_as(C.POINTER(C.c_int64)),
                                conds.ctypes.data_as(C.POINTER(C.c_double)), nn)
        z_cond = {int(nodes[i]): float(conds[i]) for i in range(cnt)}
        fb = np.zeros(nn, np.int64)
        nfb = lib.ks_get_fallback_nodes(self._h, fb.ctypes.data_as(C.POINTER(C.c_int64)), nn)
        fallback_nodes = sorted(int(v) for v in fb[:nfb])
        warnings = [  # solver.py:183-188
            f"node {nid}: Z condition estimate {c:.3e} exceeds {_COND_WARN:.0e}; results may lose accuracy"
            for nid, c in sorted(z_cond.items()) if c > _COND_WARN
        ]
        return {
            "cholesky_fallbacks": len(fallback_nodes),
            "fallback_nodes": fallback_nodes,
            "z_cond": z_cond,
            "warnings": warnings,
        }

    # parity-debugging views (the reference's leaf_factors / node_factors)
    def node_h(self, node: int) -> np.ndarray:
        r = int(self.problem.rank[node])
        out = np.zeros((r, r))
        rc = _lib.load().ks_get_node_h(self.handle, int(node), out.ctypes.data_as(C.POINTER(C.c_double)))
        if rc:
            _raise(rc)
        return out

    def leaf_factor(self, node: int) -> np.ndarray:
        m = int(self.problem.node_end[node] - self.problem.node_begin[node])
        out = np.zeros((m, m))
        rc = _lib.load().ks_get_leaf_factor(self.handle, int(node), out.ctypes.data_as(C.POINTER(C.c_double)))
        if rc:
            _raise(rc)
        return out

    def device_bytes(self) -> int:
        return int(_lib.load().ks_device_bytes(self.handle))

    def refactorize(self, lam: float, stream: int = 0) -> None:
        """Re-run the factorization on the resident inputs (device-only timing)."""
        lam = _check_lam(lam)
        rc = _lib.load().ks_factorize(self.handle, lam, C.c_void_p(stream or None))
        if rc:
            _raise(rc, self._h)
        self.lam = lam
        self.diagnostics = self._read_diagnostics()

    def set_profiling(self, on: bool) -> None:
        _lib.load().ks_set_profiling(self.handle, 1 if on else 0)

    def phase_ms(self) -> list[float]:
        ms = (C.c_double * 6)()
        n = _lib.load().ks_get_phase_ms(self.handle, ms, 6)
        return [float(ms[i]) for i in range(n)]

    def level_ms(self) -> list[float]:
        ms = (C.c_double * 64)()
        n = _lib.load().ks_get_level_ms(self.handle, ms, 64)
        return [float(ms[i]) for i in range(n)]

    def pipelined_levels(self) -> tuple[int, int]:
        """(levels planned to run per subtree on the subtree's own stream, the same
        if subtree pipelining is enabled for this handle, else 0)."""
        out = (C.c_int * 2)()
        _lib.load().ks_pipelined_levels(self.handle, out)
        return int(out[0]), int(out[1])

    def trace_report(self) -> str:
        buf = C.create_string_buffer(1 << 16)
        _lib.load().ks_trace_report(self.handle, buf, len(buf))
        return buf.value.decode()

    def last_launches(self, which: int) -> int:
        return int(_lib.load().ks_last_launches(self.handle, which))

    def close(self) -> None:
        if self._h:
            _lib.load().ks_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _check_lam(lam) -> float:
    lam = float(lam)
    if not np.isfinite(lam) or lam < 0.0:  # solver.py:101-103
        raise InvalidArgumentError(f"need lambda >= 0 and finite, got {lam}")
    return lam


def factorize(ck, lam: float, threads: int = 1, *, device: int | None = None) -> GpuHierFactor:
    """Bottom-up recursive Woodbury factorization of K~ + lam*I on the GPU.

    Mirrors kernelsolve.factorize (solver.py:92-189): lam >= 0 and finite;
    Cholesky on each leaf block with an LU fallback recorded in the
    diagnostics; a Z condition estimate above 1e14 raises
    IllConditionedError, above 1e10 it is recorded as a warning.
    """
    lam = _check_lam(lam)
    del threads  # accepted for compatibility; results do not depend on it
    prob = as_problem(ck)
    lib = _lib.load()
    dev = _default_device() if device is None else int(device)
    cprob = prob.to_c()
    h = C.c_void_p()
    rc = lib.ks_create(C.byref(cprob), dev, C.byref(h))
    if rc:
        _raise(rc)
    rc = lib.ks_factorize(h, lam, None)
    if rc:
        try:
            _raise(rc, h)
        finally:
            lib.ks_destroy(h)
    return GpuHierFactor(ck, prob, lam, h.value, dev)


def solve(hf: GpuHierFactor, b):
    """Apply (K~ + lam*I)^-1 to one vector in tree (perm) order (solver.py:192)."""
    if _is_torch_cuda(b):
        if b.dim() != 1:
            raise InvalidArgumentError(f"expected a vector, got shape {tuple(b.shape)}")
        return solve_many(hf, b[:, None])[:, 0]
    b = np.asarray(b, dtype=np.float64)
    if b.ndim != 1:
        raise InvalidArgumentError(f"expected a vector, got shape {b.shape}")
    return solve_many(hf, b[:, None])[:, 0]


def solve_many(hf: GpuHierFactor, B):
    """Apply (K~ + lam*I)^-1 to q right-hand sides at once (solver.py:200).

    Accepts a numpy array (host path: H2D, solve, D2H inside the call) or a
    torch CUDA float64 tensor (device-resident path, result on the device).
    """
    if _is_torch_cuda(B):
        return _solve_many_torch(hf, B)
    B = np.asarray(B, dtype=np.float64)
    if B.ndim != 2:
        raise InvalidArgumentError(f"expected an n x q matrix, got shape {B.shape}")
    if B.shape[0] != hf.n:
        raise InvalidArgumentError(f"right-hand side has {B.shape[0]} rows, need {hf.n}")
    if B.shape[1] == 0:
        return np.empty_like(B)
    Bc = np.ascontiguousarray(B)
    X = _host_result(Bc.shape)
    rc = _lib.load().ks_solve(hf.handle, Bc.ctypes.data_as(C.c_void_p), X.ctypes.data_as(C.c_void_p),
                              Bc.shape[1], None)
    if rc:
        _raise(rc)
    return X


def hss_matvec(hf: GpuHierFactor, w):
    """K~ @ w for the factor's compressed operator (compress.py:352-411): a
    length-n vector or an n x q matrix in tree order, numpy or CUDA torch."""
    if _is_torch_cuda(w):
        import torch

        W = w[:, None] if w.dim() == 1 else w
        if W.shape[0] != hf.n:
            raise InvalidArgumentError(f"vector length {W.shape[0]} != n = {hf.n}")
        W = W.contiguous().to(torch.float64)
        Y = torch.empty_like(W)
        stream = torch.cuda.current_stream(W.device).cuda_stream
        rc = _lib.load().ks_matvec(hf.handle, C.c_void_p(W.data_ptr()), C.c_void_p(Y.data_ptr()), W.shape[1],
                                   C.c_void_p(stream))
        if rc:
            _raise(rc)
        return Y[:, 0] if w.dim() == 1 else Y
    w = np.asarray(w, dtype=np.float64)
    if w.shape[0] != hf.n:
        raise InvalidArgumentError(f"vector length {w.shape[0]} != n = {hf.n}")
    W = np.ascontiguousarray(w[:, None] if w.ndim == 1 else w)
    Y = _host_result(W.shape)
    rc = _lib.load().ks_matvec(hf.handle, W.ctypes.data_as(C.c_void_p), Y.ctypes.data_as(C.c_void_p), W.shape[1], None)
    if rc:
        _raise(rc)
    return Y[:, 0] if w.ndim == 1 else Y


def release_cached_memory(device: int | None = None) -> None:
    """Return the device memory the library caches between handles (its private
    stream-ordered pool keeps up to KS_POOL_GB, default 32 GB, of freed factor
    storage for the next factorize) to the driver, like torch.cuda.empty_cache."""
    dev = _default_device() if device is None else int(device)
    rc = _lib.load().ks_trim_pool(dev)
    if rc:
        _raise(rc)


_PINNED_RESULT_MAX = 1 << 28  # results up to 256 MB come back in page-locked memory


def _host_result(shape) -> np.ndarray:
    """A fresh float64 host array for a result the library copies out of the
    device. Page-locked (torch's caching pinned allocator, so repeated solves
    reuse the blocks): the D2H copy is then one DMA into the caller's array
    instead of a staged copy into fresh pageable pages (config 3, q = 1: 6.3 ->
    5.2 ms per host solve). Larger results use ordinary memory."""
    nbytes = 8 * int(np.prod(shape))
    if 0 < nbytes <= _PINNED_RESULT_MAX:
        try:
            import torch

            return torch.empty(tuple(int(x) for x in shape), dtype=torch.float64, pin_memory=True).numpy()
        except Exception:  # no torch / no pinned memory left: pageable is still correct
            pass
    return np.empty(shape, dtype=np.float64)


def _is_torch_cuda(x) -> bool:
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


def _solve_many_torch(hf: GpuHierFactor, B):
    import torch

    if B.dim() != 2:
        raise InvalidArgumentError(f"expected an n x q matrix, got shape {tuple(B.shape)}")
    if B.shape[0] != hf.n:
        raise InvalidArgumentError(f"right-hand side has {B.shape[0]} rows, need {hf.n}")
    if B.dtype != torch.float64:
        raise InvalidArgumentError("right-hand side must be float64")
    if B.shape[1] == 0:
        return torch.empty_like(B)
    Bc = B.contiguous()
    X = torch.empty_like(Bc)
    stream = torch.cuda.current_stream(Bc.device).cuda_stream
    rc = _lib.load().ks_solve(hf.handle, C.c_void_p(Bc.data_ptr()), C.c_void_p(X.data_ptr()), Bc.shape[1],
                              C.c_void_p(stream))
    if rc:
        _raise(rc)
    return X
