"""Rank program for tests/test_launch_cpu.py, started by
paper_1602_01376_b200.launch.spawn (torchrun, gloo on CPU). Runs the real
sharded orchestration with the CPU oracle backend per rank.

argv: case out_path [fail_rank]   (fail_rank: that rank's local factorization
raises IllConditionedError(node 3, 1e15); every rank must raise it, none hangs)
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

from conftest import load_golden  # noqa: E402
from shard_oracle import OracleShard  # noqa: E402

from paper_1602_01376_b200 import distributed as kd  # noqa: E402
from paper_1602_01376_b200 import errors as E  # noqa: E402
from paper_1602_01376_b200.problem import from_arrays  # noqa: E402


def main():
    case, out = sys.argv[1], sys.argv[2]
    fail_rank = int(sys.argv[3]) if len(sys.argv) > 3 else -1
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    g = load_golden(case)
    root, peers = kd.shard_for(from_arrays(g), world, rank)
    sh = OracleShard(g, root, peers)
    if rank == fail_rank:
        def boom(lam):
            raise E.IllConditionedError(3, 1e15)
        sh.factorize = boom
    res = {"rank": rank, "world": world, "env_world": os.environ.get("WORLD_SIZE")}
    try:
        kd.factorize_sharded(sh, float(g["lam"]))
        X = kd.solve_many_sharded(sh, torch.from_numpy(g["b"]))
        res["err"] = float(np.linalg.norm(X.numpy() - g["u"]) / np.linalg.norm(g["u"]))
    except E.KernelSolveError as exc:
        res["raised"] = type(exc).__name__
        res["node_id"] = getattr(exc, "node_id", None)
    with open(f"{out}.{rank}.json", "w") as fh:
        json.dump(res, fh)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
