"""Multi-GPU factor/solve by subtree sharding (north_star).

One process per GPU. With p = 2^k ranks, rank g owns node `peers[g]` at tree
level k (BFS order = left to right = its contiguous slice of tree order): it
factors that subtree alone, then the ranks all-gather the p skeleton-sized
reduced matrices H (s x s each) and every rank redundantly factors the k top
levels. The solve mirrors it: local up pass -> all-gather of the p skeleton
weight blocks c (s x q) -> redundant top up/down pass -> local down pass. No
other data crosses GPUs; the exchange is NCCL all-gather over NVLink when the
process group is NCCL (gloo in the CPU tests).

The orchestration functions take a per-rank backend object:
`LibShard` drives libinvaskit.so (ks_create_shard & co., include/invaskit.h);
tests substitute a CPU oracle backend with the same methods.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib
from .problem import Problem, as_problem
from .solver import _check_lam, _raise


def level_nodes(prob: Problem, level: int) -> list[int]:
    lev = prob.node_level()
    return [int(v) for v in np.flatnonzero(lev == level)]


def shard_for(prob: Problem, world: int, rank: int) -> tuple[int, list[int]]:
    """Shard root of `rank` and the ordered list of all shard roots."""
    k = int(round(np.log2(world)))
    if 2 ** k != world:
        raise ValueError(f"world size must be a power of two, got {world}")
    peers = level_nodes(prob, k)
    if len(peers) != world:
        raise ValueError(f"tree has {len(peers)} nodes at level {k}, need {world}")
    peers.sort(key=lambda v: int(prob.node_begin[v]))
    return peers[rank], peers


class LibShard:
    """libinvaskit.so sharded handle on one GPU."""

    def __init__(self, ck, shard_root: int, device: int):
        import torch

        self.torch = torch
        self.prob = as_problem(ck)
        self.device = device
        self.lib = _lib.load()
        cp = self.prob.to_c()
        h = C.c_void_p()
        rc = self.lib.ks_create_shard(C.byref(cp), device, int(shard_root), C.byref(h))
        if rc:
            _raise(rc)
        self.h = h.value
        info = np.zeros(64 + self.prob.n_nodes, np.int64)
        n = self.lib.ks_shard_info(self.h, info.ctypes.data_as(C.POINTER(C.c_int64)), info.size)
        self.shard_root, self.level, self.begin, self.end, self.s_pad, npeer = (int(x) for x in info[:6])
        self.peers = [int(x) for x in info[6:6 + npeer]]
        assert n == 6 + npeer
        self.dev = torch.device("cuda", device)

    def _stream(self):
        return C.c_void_p(self.torch.cuda.current_stream(self.dev).cuda_stream)

    def _chk(self, rc):
        if rc:
            _raise(rc, self.h)

    def factorize(self, lam: float) -> None:
        self._chk(self.lib.ks_factorize(self.h, float(lam), self._stream()))

    def export_h(self, node: int):
        t = self.torch.empty(self.s_pad, self.s_pad, dtype=self.torch.float64, device=self.dev)
        self._chk(self.lib.ks_node_exchange(self.h, 0, node, C.c_void_p(t.data_ptr()), 0, 0, self._stream()))
        return t

    def import_h(self, node: int, t) -> None:
        self._chk(self.lib.ks_node_exchange(self.h, 0, node, C.c_void_p(t.data_ptr()), 0, 1, self._stream()))

    def factorize_top(self) -> None:
        self._chk(self.lib.ks_factorize_top(self.h, self._stream()))

    def solve_up(self, B_local) -> None:
        B_local = B_local.to(self.dev, dtype=self.torch.float64).contiguous()
        self._B = B_local
        self._chk(self.lib.ks_solve_up(self.h, C.c_void_p(B_local.data_ptr()), B_local.shape[1], self._stream()))

    def export_c(self, node: int, q: int):
        t = self.torch.empty(self.s_pad, q, dtype=self.torch.float64, device=self.dev)
        self._chk(self.lib.ks_node_exchange(self.h, 1, node, C.c_void_p(t.data_ptr()), q, 0, self._stream()))
        return t

    def import_c(self, node: int, t) -> None:
        q = t.shape[1]
        self._chk(self.lib.ks_node_exchange(self.h, 1, node, C.c_void_p(t.data_ptr()), q, 1, self._stream()))

    def solve_top(self, q: int) -> None:
        self._chk(self.lib.ks_solve_top(self.h, q, self._stream()))

    def solve_down(self, q: int):
        X = self.torch.empty(self.end - self.begin, q, dtype=self.torch.float64, device=self.dev)
        self._chk(self.lib.ks_solve_down(self.h, C.c_void_p(X.data_ptr()), q, self._stream()))
        return X

    def close(self) -> None:
        if self.h:
            self.lib.ks_destroy(self.h)
            self.h = None


# ---------------------------------------------------------------------------
# orchestration (backend-agnostic)
# ---------------------------------------------------------------------------
def _err_info(exc: BaseException) -> tuple:
    from . import errors as E

    if isinstance(exc, E.IllConditionedError):
        return ("IllConditionedError", int(exc.node_id), float(exc.cond_estimate))
    return (type(exc).__name__, str(exc))


def _rebuild(info: tuple, rank: int) -> BaseException:
    from . import errors as E

    name = info[0]
    if name == "IllConditionedError":
        return E.IllConditionedError(info[1], info[2])
    cls = getattr(E, name, None)
    msg = f"rank {rank}: {info[1]}"
    if isinstance(cls, type) and issubclass(cls, Exception) and name != "IllConditionedError":
        return cls(msg)
    return E.KernelSolveError(f"rank {rank} failed with {name}: {info[1]}")


def _agree(exc: BaseException | None, group=None) -> None:
    """Collective status check before an exchange: if any rank failed in its
    local phase, every rank raises the first failing rank's error (same type,
    same node id / condition estimate) instead of blocking in the collective."""
    import torch
    import torch.distributed as dist

    nccl = dist.get_backend(group) == "nccl"
    flag = torch.tensor([0 if exc is None else 1], dtype=torch.int32,
                        device=torch.device("cuda", torch.cuda.current_device()) if nccl else "cpu")
    dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
    if int(flag.item()) == 0:
        return
    infos = [None] * dist.get_world_size(group)
    dist.all_gather_object(infos, None if exc is None else _err_info(exc), group=group)
    first = next(r for r, i in enumerate(infos) if i is not None)
    if exc is not None and first == dist.get_rank(group):
        raise exc
    raise _rebuild(infos[first], first) from exc


def factorize_sharded(backend, lam: float, group=None) -> None:
    """Local subtree factorization, all-gather of the level-k H blocks, top levels.
    A failure on any rank (e.g. IllConditionedError inside one subtree) is
    raised on every rank (no rank is left waiting in the all-gather)."""
    import torch.distributed as dist

    lam = _check_lam(lam)
    err = None
    try:
        backend.factorize(lam)
    except Exception as e:  # noqa: BLE001 -- re-raised on every rank by _agree
        err = e
    _agree(err, group)
    H = backend.export_h(backend.shard_root)
    world = len(backend.peers)
    Hs = [H.new_empty(H.shape) for _ in range(world)]
    dist.all_gather(Hs, H, group=group)
    for node, Hn in zip(backend.peers, Hs):
        if node != backend.shard_root:
            backend.import_h(node, Hn)
    backend.factorize_top()


def solve_many_sharded(backend, B, group=None, gather: bool = True):
    """Solve with the sharded factor. B: (n, q) tree order (torch tensor, any
    device) or the shard's own rows if gather is False. Returns the full X
    (all-gathered to every rank) or the local rows.

    The subtree-root block c travels with one status row: a rank whose local
    up pass failed still takes part in the all-gather (no rank blocks), and
    after the down pass every rank raises that rank's error."""
    import torch
    import torch.distributed as dist

    if B.dim() != 2:
        raise ValueError("B must be n x q")
    q = B.shape[1]
    B_local = B[backend.begin:backend.end] if gather else B
    err = None
    try:
        backend.solve_up(B_local)
        c = backend.export_c(backend.shard_root, q)
    except Exception as e:  # noqa: BLE001 -- re-raised on every rank below
        err = e
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
        c = torch.zeros(backend.s_pad, q, dtype=torch.float64, device=dev)
    cst = torch.cat([c, c.new_full((1, q), 0.0 if err is None else 1.0)], dim=0)
    world = len(backend.peers)
    cs = [cst.new_empty(cst.shape) for _ in range(world)]
    dist.all_gather(cs, cst, group=group)
    status = torch.stack([x[-1, 0] for x in cs])
    X_local = None
    if err is None:
        for node, cn in zip(backend.peers, cs):
            if node != backend.shard_root:
                backend.import_c(node, cn[:-1].contiguous())
        backend.solve_top(q)
        X_local = backend.solve_down(q)
    if float(status.max()) > 0.0:  # one host read per solve, after the device work is queued
        _agree(err if err is not None else None, group)
    if not gather:
        return X_local
    sizes = [None] * world
    dist.all_gather_object(sizes, int(X_local.shape[0]), group=group)
    mx = max(sizes)
    pad = X_local.new_zeros(mx, q)
    pad[: X_local.shape[0]] = X_local
    parts = [pad.new_empty(mx, q) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:sz] for p, sz in zip(parts, sizes)], dim=0)


# ---------------------------------------------------------------------------
# public multi-GPU entry points (one process per GPU, torch.distributed)
# ---------------------------------------------------------------------------
class ShardedFactor:
    """The subtree-sharded factor of one rank: `solve_many` is collective
    (every rank calls it with the same B), and returns the full solution on
    every rank (gather=True) or the rank's own rows of it."""

    def __init__(self, backend, lam: float, group=None):
        self.backend = backend
        self.lam = lam
        self.group = group

    @property
    def rows(self) -> tuple[int, int]:
        return self.backend.begin, self.backend.end

    def solve_many(self, B, gather: bool = True):
        return solve_many_sharded(self.backend, B, self.group, gather)

    def close(self) -> None:
        self.backend.close()


def factorize_distributed(ck, lam: float, threads: int = 1, *, group=None, device: int | None = None) -> ShardedFactor:
    """factorize (solver.py:92) over the ranks of `group`: rank g factors the
    g-th subtree at level log2(world) and the top levels redundantly. Every
    rank must call it; an error on any rank is raised on all of them."""
    import torch.distributed as dist

    del threads
    lam = _check_lam(lam)
    prob = as_problem(ck)
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    root, _ = shard_for(prob, world, rank)
    dev = int(os.environ.get("LOCAL_RANK", "0")) if device is None else int(device)
    err, sh = None, None
    try:
        sh = LibShard(prob, root, dev)
    except Exception as e:  # noqa: BLE001 -- re-raised on every rank by _agree
        err = e
    _agree(err, group)
    try:
        factorize_sharded(sh, lam, group)
    except Exception:
        sh.close()
        raise
    return ShardedFactor(sh, lam, group)
