"""The N-rank launcher bench.py uses (paper_1602_01376_b200.launch: torchrun
on 127.0.0.1), driven end to end on CPU with gloo: ranks start, find each
other, run the sharded orchestration, and a failure on one rank surfaces on
every rank instead of leaving the others blocked in a collective."""
import json
import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _run(tmp_path, world, case, fail_rank=None):
    from paper_1602_01376_b200 import launch
    out = str(tmp_path / "res")
    args = [case, out] + ([str(fail_rank)] if fail_rank is not None else [])
    r = launch.spawn(world, os.path.join(HERE, "_launch_worker.py"), args, timeout=300, capture=True)
    assert r.returncode == 0, r.stderr[-3000:]
    return [json.load(open(f"{out}.{k}.json")) for k in range(world)]


@pytest.mark.parametrize("world", [2, 4])
def test_launcher_runs_sharded_solve(tmp_path, world):
    res = _run(tmp_path, world, "cfg1")
    assert sorted(r["rank"] for r in res) == list(range(world))
    for r in res:
        assert r["world"] == world and r["env_world"] == str(world)
        assert r["err"] <= 1e-12, r


def test_failure_on_one_rank_raises_everywhere(tmp_path):
    res = _run(tmp_path, 2, "cfg1", fail_rank=1)
    for r in res:
        assert r["raised"] == "IllConditionedError" and r["node_id"] == 3, r


def test_bench_spawns_ranks_when_not_launched(monkeypatch):
    """bench.py --gpus N without WORLD_SIZE re-launches itself as N ranks."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_1602_01376_b200 import launch
    calls = []

    class R:
        returncode = 0

    monkeypatch.setattr(launch, "spawn", lambda n, script, args, env=None: calls.append((n, script, args, env)) or R())
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    with pytest.raises(SystemExit) as ei:
        bench.main()
    assert ei.value.code == 0
    n, script, args, env = calls[0]
    assert n == 4 and script.endswith("bench.py") and args == ["--gpus", "4", "--steps", "2"]
    assert env["NCCL_DEBUG"] == "INFO"
    argv = launch.torchrun_argv(4, script, args, port=12345)
    assert "--nproc-per-node=4" in argv and "--master-addr=127.0.0.1" in argv
