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
def factorize_sharded(backend, lam: float, group=None) -> None:
    """Local subtree factorization, all-gather of the level-k H blocks, top levels."""
    import torch.distributed as dist

    lam = _check_lam(lam)
    backend.factorize(lam)
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
    (all-gathered to every rank) or the local rows."""
    import torch
    import torch.distributed as dist

    if B.dim() != 2:
        raise ValueError("B must be n x q")
    q = B.shape[1]
    B_local = B[backend.begin:backend.end] if gather else B
    backend.solve_up(B_local)
    c = backend.export_c(backend.shard_root, q)
    world = len(backend.peers)
    cs = [c.new_empty(c.shape) for _ in range(world)]
    dist.all_gather(cs, c, group=group)
    for node, cn in zip(backend.peers, cs):
        if node != backend.shard_root:
            backend.import_c(node, cn)
    backend.solve_top(q)
    X_local = backend.solve_down(q)
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
# bench.py --gpus N (torchrun): strong scaling of config 3 over N GPUs
# ---------------------------------------------------------------------------
def bench_main(args, metric: str) -> None:
    import json
    import time

    import torch
    import torch.distributed as dist

    from . import yardstick
    from .configs import CONFIGS

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from producer import make_operator, make_rhs

    cfg = CONFIGS[args.config]
    op = make_operator(cfg, device="cuda")
    # identical operator bits on every rank: rank 0's P wins
    coeff = torch.from_numpy(op["coeff"]).cuda()
    dist.broadcast(coeff, 0)
    op["coeff"] = coeff.cpu().numpy()
    del coeff
    prob = as_problem(op)
    root, peers = shard_for(prob, world, rank)
    sh = LibShard(prob, root, local)
    b = torch.from_numpy(make_rhs(cfg, op["perm"], 1)).cuda()
    F = yardstick.factor_flops(op)
    for _ in range(args.warmup):
        factorize_sharded(sh, cfg.lam)
        solve_many_sharded(sh, b, gather=False)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    dist.barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        ev[i][0].record()
        factorize_sharded(sh, cfg.lam)
        ev[i][1].record()
        solve_many_sharded(sh, b, gather=False)
        ev[i][2].record()
    torch.cuda.synchronize()
    dist.barrier()
    tf = float(np.mean([e[0].elapsed_time(e[1]) for e in ev]))
    ts = float(np.mean([e[1].elapsed_time(e[2]) for e in ev]))
    t = torch.tensor([tf, ts], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tf, ts = float(t[0]), float(t[1])
    if rank == 0:
        line = {
            "metric": metric, "value": F / (tf * 1e-3) / 1e12, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tf + ts, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{cfg.name} factor+solve q=1, subtree-sharded", "n": cfg.n, "d": cfg.d,
                       "leaf": cfg.leaf_size, "rank": cfg.max_rank, "parallelism": f"subtree{world}"},
            "factor_ms": tf, "solve_ms": ts,
        }
        print(json.dumps(line), flush=True)
    sh.close()
    dist.destroy_process_group()
