"""Device timeline of one factorization (graph replay) and one solve, from
CUPTI activity records (torch.profiler): every kernel of libinvaskit with its
stream, start and end. Prints a per-kernel-name summary (total busy time,
launches), the concurrency profile (how much of the step each number of
concurrently running kernels covers), and per-phase windows; writes the raw
records as JSON for offline analysis.

    python tools/timeline.py [--config cfg3] [--out gpurun_out/timeline.json] [--what factor|solve|both]
"""
import argparse
import json
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1602_01376_b200 as ks  # noqa: E402
from paper_1602_01376_b200.configs import CONFIGS  # noqa: E402
from producer import make_operator, make_rhs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--q", type=int, default=1)
ap.add_argument("--what", default="both", choices=["both", "factor", "solve"])
ap.add_argument("--out", default="gpurun_out/timeline.json")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--e2e", action="store_true", help="profile the public-API factorize from pinned host memory (uploads included)")
a = ap.parse_args()
cfg = CONFIGS[a.config]
op = make_operator(cfg)
if a.e2e:
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
    from bench import _pinned_problem

    torch.cuda.empty_cache()
    pin, _ = _pinned_problem(torch, op)
    pprob = ks.from_arrays(pin)
    h0 = ks.factorize(pprob, cfg.lam)  # warm the pool
    h0.close()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        h1 = ks.factorize(pprob, cfg.lam)
        torch.cuda.synchronize()
    recs = []
    for e in prof.events():
        if e.device_type.name != "CUDA":
            continue
        tr = e.time_range
        recs.append({"name": e.name, "start": tr.start, "end": tr.end,
                     "stream": getattr(e, "device_resource_id", None) or getattr(e, "thread", 0)})
    recs = [r for r in recs if r["end"] > r["start"]]
    recs.sort(key=lambda r: r["start"])
    t0 = recs[0]["start"]
    print(f"e2e span {(max(r['end'] for r in recs) - t0) / 1e3:.3f} ms, {len(recs)} records")
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump({"t0": t0, "records": recs}, fh)
    sys.exit(0)
hf = ks.factorize(ks.from_arrays(op), cfg.lam)
B = torch.from_numpy(make_rhs(cfg, op["perm"], a.q)).cuda()
for _ in range(2):
    hf.refactorize(cfg.lam)
    ks.solve_many(hf, B)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(a.reps):
        if a.what in ("both", "factor"):
            hf.refactorize(cfg.lam)
        if a.what in ("both", "solve"):
            ks.solve_many(hf, B)
    torch.cuda.synchronize()

recs = []
for e in prof.events():
    if e.device_type.name != "CUDA":
        continue
    tr = e.time_range
    recs.append({"name": e.name, "start": tr.start, "end": tr.end,
                 "stream": getattr(e, "device_resource_id", None) or getattr(e, "thread", 0)})
recs = [r for r in recs if r["end"] > r["start"]]
recs.sort(key=lambda r: r["start"])
t0 = recs[0]["start"]
t1 = max(r["end"] for r in recs)
print(f"span {(t1 - t0) / 1e3:.3f} ms, {len(recs)} kernels/copies")
agg = defaultdict(lambda: [0, 0.0])
for r in recs:
    nm = r["name"].split("(")[0][:60]
    agg[nm][0] += 1
    agg[nm][1] += (r["end"] - r["start"]) / 1e3
print("busy ms  launches  kernel")
for nm, (c, ms) in sorted(agg.items(), key=lambda x: -x[1][1])[:40]:
    print(f"{ms:8.3f} {c:8d}  {nm}")
# concurrency profile: time covered by exactly k running kernels
ev = []
for r in recs:
    ev.append((r["start"], 1))
    ev.append((r["end"], -1))
ev.sort()
cover = defaultdict(float)
k, last = 0, ev[0][0]
for t, d in ev:
    cover[k] += t - last
    k += d
    last = t
print("concurrency: " + ", ".join(f"{kk}:{v / 1e3:.2f}ms" for kk, v in sorted(cover.items())))
# streams
by_stream = defaultdict(lambda: [0, 0.0, 1e30, 0.0])
for r in recs:
    s = by_stream[r["stream"]]
    s[0] += 1
    s[1] += (r["end"] - r["start"]) / 1e3
    s[2] = min(s[2], r["start"])
    s[3] = max(s[3], r["end"])
for sid, (c, ms, a0, a1) in sorted(by_stream.items(), key=lambda x: x[1][2]):
    print(f"stream {sid}: {c} launches, busy {ms:.2f} ms, window {(a0 - t0) / 1e3:.2f}-{(a1 - t0) / 1e3:.2f} ms")
os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
with open(a.out, "w") as fh:
    json.dump({"t0": t0, "records": recs}, fh)
print("wrote", a.out)
