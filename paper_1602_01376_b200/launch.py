"""One process per GPU: start N ranks of a command with torch.distributed.run
(torchrun) on this node, rendezvous on 127.0.0.1.

`bench.py --gpus N` uses it when it is not already running under a launcher
(no WORLD_SIZE in the environment), so `python bench.py --gpus 8` runs the
subtree-sharded factor/solve on 8 GPUs by itself. The launched command sees
RANK / LOCAL_RANK / WORLD_SIZE / MASTER_ADDR / MASTER_PORT as usual.
"""

from __future__ import annotations

import os
import socket
import subprocess
import sys


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def under_launcher() -> bool:
    return "WORLD_SIZE" in os.environ and "RANK" in os.environ


def torchrun_argv(nproc: int, script: str, args: list[str], port: int | None = None) -> list[str]:
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={int(nproc)}",
            "--master-addr=127.0.0.1", f"--master-port={port or free_port()}", script, *args]


def spawn(nproc: int, script: str, args: list[str], env: dict | None = None, timeout: float | None = None,
          capture: bool = False) -> subprocess.CompletedProcess:
    """Run `script args` as nproc ranks; returns the launcher's completed process
    (rank outputs go to this process's stdout/stderr unless capture=True)."""
    if nproc < 1:
        raise ValueError(f"need at least one rank, got {nproc}")
    e = dict(os.environ)
    for k in ("RANK", "LOCAL_RANK", "WORLD_SIZE", "LOCAL_WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT",
              "GROUP_RANK", "ROLE_RANK", "TORCHELASTIC_RUN_ID"):
        e.pop(k, None)
    e.setdefault("OMP_NUM_THREADS", "1")
    if env:
        e.update(env)
    return subprocess.run(torchrun_argv(nproc, script, args), env=e, timeout=timeout, capture_output=capture,
                          text=True)
