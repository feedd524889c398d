"""Benchmark: Inv-ASKIT factorization TFLOP/s (fp64) + solve time at BASELINE config 3
(N = 1,048,576, d = 28, m = 1024, s = 256, h = 1.5, lambda = 0.1) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg3]

One step = one factorization of K~ + lambda I (kernelsolve.factorize,
solver.py:92-189) plus one solve with q = 1 (solve_many, solver.py:200-237),
inputs resident in HBM (`value`); `e2e` runs the same step through the public
Python API from pinned host buffers (operator upload + factor + solve + result
read back). The operator inputs (tree, skeletons, P) are produced on the box by
`producer` (not timed). `--impl reference` times the CPU oracle port of the
reference algorithm (oracle/ks_oracle.py) on a bounded sample of the same
workload. Prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "factorization TFLOP/s fp64 + solve time (N=1M, d=28) at 1/2/4/8 B200 vs CPU"


def _peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, interval_ms: int = 20):
        self.index = index
        self.interval = interval_ms
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", str(self.interval)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.rows = []
        if self.proc is None:
            return False
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 8:
                self.rows.append(parts)
        return False

    def summary(self) -> dict:
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def measure_fp64_sustained(torch, seconds: float = 3.0) -> float:
    """cuBLAS DGEMM 8192^3 back to back for `seconds` (power-capped clocks)."""
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = a @ b
    torch.cuda.synchronize()
    reps, t0 = 0, time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.perf_counter() - t0 < seconds:
        for _ in range(8):
            torch.matmul(a, b, out=c)
        reps += 8
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    del a, b, c
    torch.cuda.empty_cache()
    return 2.0 * n ** 3 * reps / (ms * 1e-3) / 1e12


def measure_fp64_peak(torch) -> float:
    """cuBLAS DGEMM 8192^3, best of 10 (the fp64 peak is not in MEASURED_PEAKS.json)."""
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    a @ b
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    torch.cuda.empty_cache()
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


# ---------------------------------------------------------------------------
# CPU: the oracle port of the reference algorithm on a bounded sample
# ---------------------------------------------------------------------------
def cpu_sample(repeats: int = 1) -> dict:
    """Reference algorithm (oracle/ks_oracle.py restatement, numpy + the box's
    BLAS threads) on the cfg3-shaped golden operator (reference inputs, N=4096:
    4 leaves of m=1024, s=256, d=28). Factor TFLOP/s is measured; the full-size
    recursive solve (4^10 leaf solves at N=1M) is extrapolated
    from the sample's 4^2, and the O(N) telescoping CPU solve linearly."""
    from oracle import ks_oracle as O
    from paper_1602_01376_b200 import yardstick

    with np.load(os.path.join(ROOT, "tests", "golden", "cfg3s.npz")) as z:
        g = {k: z[k] for k in z.files}
    prob = O.Problem(g)
    lam = float(g["lam"])
    b = g["b"][:, :1]
    tf, ts, tt = [], [], []
    for _ in range(repeats):
        t0 = time.perf_counter()
        of = O.factorize(prob, lam)
        t1 = time.perf_counter()
        O.solve_many_recursive(of, b)
        t2 = time.perf_counter()
        O.solve_many_telescoping(of, b)
        t3 = time.perf_counter()
        tf.append(t1 - t0)
        ts.append(t2 - t1)
        tt.append(t3 - t2)
    F = yardstick.factor_flops(g)
    tf_m, ts_m, tt_m = float(np.median(tf)), float(np.median(ts)), float(np.median(tt))
    leaves_sample, leaves_full = 4, 1024
    return {
        "factor_tflops": F / tf_m / 1e12,
        "factor_s_sample": tf_m,
        "solve_ms_extrapolated": ts_m * (leaves_full / leaves_sample) ** 2 * 1e3,
        "solve_telescoping_ms_extrapolated": tt_m * (leaves_full / leaves_sample) * 1e3,
        "cores": os.cpu_count(),
        "sample": "cfg3-shaped reference operator N=4096 (4 leaves m=1024, 3 internal s=256, d=28): "
                  "factorize measured; recursive solve extrapolated x(1024/4)^2 leaf solves, "
                  "telescoping solve x(1024/4)",
    }


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    steps = []
    for _ in range(args.warmup and 1):
        cpu_sample(1)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        steps.append(cpu_sample(1))
    wall = time.perf_counter() - t0
    val = float(np.median([s["factor_tflops"] for s in steps]))
    solve_ms = float(np.median([s["solve_ms_extrapolated"] for s in steps]))
    s0 = steps[0]
    line = {
        "metric": METRIC, "value": val, "unit": "TFLOP/s", "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall / max(args.steps, 1) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg3 factor+solve (bounded CPU sample)", "n": 1048576, "d": 28, "leaf": 1024,
                   "rank": 256, "h": 1.5, "lambda": 0.1, "q": 1},
        "solve_ms": solve_ms,
        "solve_telescoping_ms": float(np.median([s["solve_telescoping_ms_extrapolated"] for s in steps])),
        "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": s0["cores"], "kind": "port", "sample": s0["sample"]},
        "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU
# ---------------------------------------------------------------------------
def _pinned_problem(torch, op: dict) -> tuple[dict, int]:
    """Copy the operator's arrays into pinned host memory (e2e H2D source)."""
    out, nbytes = {}, 0
    for k, v in op.items():
        a = np.asarray(v)
        if a.ndim == 0:
            out[k] = a
            continue
        t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
        t.numpy()[...] = a
        out[k] = t.numpy()
        if k in ("coords", "perm", "node_begin", "node_end", "node_left", "node_right", "rank", "skel_off", "skel",
                 "coeff_off", "coeff"):
            nbytes += a.nbytes
    return out, nbytes


def run_ours(args) -> None:
    import torch

    import paper_1602_01376_b200 as ks
    from paper_1602_01376_b200 import yardstick
    from paper_1602_01376_b200.configs import CONFIGS
    from producer import make_operator, make_rhs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        from paper_1602_01376_b200 import distributed as kd
        return kd.bench_main(args, METRIC)
    torch.cuda.set_device(local)
    cfg = CONFIGS[args.config]
    t0 = time.perf_counter()
    op = make_operator(cfg, device="cuda", verbose=args.verbose)
    t_prod = time.perf_counter() - t0
    prob = ks.from_arrays(op)
    ys = yardstick.summary(op, 1)
    F = ys["factor_flops"]
    q32 = 32 if 32 in cfg.q else max(cfg.q)
    b1 = make_rhs(cfg, op["perm"], 1)
    bq = make_rhs(cfg, op["perm"], q32)
    fp64_peak = measure_fp64_peak(torch)
    with Clocks(local, interval_ms=20) as clk_dgemm:
        fp64_sustained = measure_fp64_sustained(torch)
    peaks = _peaks()
    hbm_peak = float(peaks.get("hbm_gbs", 6538.9))

    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    hf = ks.factorize(prob, cfg.lam)
    B1 = torch.from_numpy(b1).cuda()
    BQ = torch.from_numpy(bq).cuda()
    for _ in range(args.warmup):
        hf.refactorize(cfg.lam, sp)
        ks.solve_many(hf, B1)
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    phases = []
    launches = 0
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        for i in range(args.steps):
            ev[i][0].record(stream)
            hf.refactorize(cfg.lam, sp)
            ev[i][1].record(stream)
            X = ks.solve_many(hf, B1)
            ev[i][2].record(stream)
            launches += hf.last_launches(0) + hf.last_launches(1)
        torch.cuda.synchronize()
    t_fac = [ev[i][0].elapsed_time(ev[i][1]) for i in range(args.steps)]
    t_sol = [ev[i][1].elapsed_time(ev[i][2]) for i in range(args.steps)]
    ms_fac, ms_sol = float(np.mean(t_fac)), float(np.mean(t_sol))
    # one extra, eager (non-graph) factorization with per-phase / per-level events
    hf.set_profiling(True)
    hf.refactorize(cfg.lam, sp)
    phases.append(hf.phase_ms())
    levels_ms = hf.level_ms()
    hf.set_profiling(False)
    # q = 32 solve (config 3 lists 1 and 32 RHS)
    ks.solve_many(hf, BQ)
    torch.cuda.synchronize()
    tq = []
    for _ in range(5):  # median of 5 single solves (robust to a stray stall)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        XQ = ks.solve_many(hf, BQ)
        e1.record(stream)
        torch.cuda.synchronize()
        tq.append(e0.elapsed_time(e1))
    ms_sol_q = float(np.median(tq))
    # residual of the benchmarked solve through the GPU compressed matvec
    # (hss_matvec, compress.py:352-411): ||(K~ + lam I) u - b|| / ||b||
    Ku = ks.hss_matvec(hf, X)
    resid = float(torch.linalg.norm(Ku + cfg.lam * X - B1) / torch.linalg.norm(B1))
    del Ku
    u = X.cpu().numpy()
    del X, XQ
    # e2e through the public API from pinned host memory
    # what the JSON line needs from the device-resident factor, then release it
    # (and torch's cached blocks) so the public-API calls below run as a user's would
    dev_bytes = hf.device_bytes()
    max_zc = max(hf.diagnostics["z_cond"].values())
    n_fallbacks = hf.diagnostics["cholesky_fallbacks"]
    hf.close()
    del hf, B1, BQ
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    pin, h2d = _pinned_problem(torch, op)
    pin_prob = ks.from_arrays(pin)
    b_pin = torch.from_numpy(b1).pin_memory().numpy()
    e2e_fac, e2e_sol = [], []
    for i in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h2 = ks.factorize(pin_prob, cfg.lam)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        u2 = ks.solve_many(h2, b_pin)
        t2 = time.perf_counter()
        h2.close()
        e2e_fac.append(t1 - t0)
        e2e_sol.append(t2 - t1)
        print(f"[bench] e2e rep {i}: factorize {1e3 * (t1 - t0):.1f} ms, solve {1e3 * (t2 - t1):.1f} ms",
              file=sys.stderr, flush=True)
    ms_e2e_fac = float(np.median(e2e_fac)) * 1e3
    ms_e2e_sol = float(np.median(e2e_sol)) * 1e3
    same = float(np.linalg.norm(u2 - u) / np.linalg.norm(u))
    ph = np.mean(np.array(phases), axis=0).tolist() if phases else []
    cpu = cpu_sample(1) if not args.no_cpu else None
    B_solve = yardstick.solve_bytes(op, 1)
    # DRAM bytes per factorization / per q=1 solve from the committed ncu capture
    # (profiles/r01_dram_traffic.json: cold caches, an upper bound), config 3 only
    traffic = {}
    tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01_dram_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            tj = json.load(fh)
        if tj.get("config") == cfg.name:
            traffic = tj
    line = {
        "metric": METRIC,
        "value": F / (ms_fac * 1e-3) / 1e12,
        "unit": "TFLOP/s",
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_fac + ms_sol,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (config-3 recipe points from the reference RNG; tree restated bit-exactly; skeletons/P by a GPU restatement of the reference ID with kNN-guided sampling)",
        "config": {"workload": f"{cfg.name} factor+solve q=1", "n": cfg.n, "d": cfg.d, "leaf": cfg.leaf_size,
                   "rank": cfg.max_rank, "h": cfg.h, "lambda": cfg.lam, "q": 1,
                   "l2": "inputs larger than L2 (factor working set %.1f GB)" % (dev_bytes / 1e9)},
        "factor_ms": ms_fac,
        "solve_ms": ms_sol,
        f"solve_ms_q{q32}": ms_sol_q,
        "factor_phase_ms_eager": {"leaves": ph[0] + ph[1] + ph[2], "internal_levels": ph[3],
                                  "total": ph[4]} if ph else None,
        "level_ms": levels_ms,
        "yardstick": {"factor_tflop": F / 1e12, "solve_gb_q1": B_solve / 1e9},
        "roofline": {"bound": "tensor", "achieved": F / (ms_fac * 1e-3) / 1e12, "peak": fp64_peak,
                     "unit": "TFLOP/s", "frac": F / (ms_fac * 1e-3) / 1e12 / fp64_peak,
                     "traffic": traffic.get("factor_bytes"), "traffic_source": traffic.get("source"),
                     "kernel": "whole factorization (DMMA GEMM + panel kernels); peak = cuBLAS DGEMM 8192^3 measured live (burst, best of 10)",
                     "peak_sustained": fp64_sustained, "frac_of_sustained": F / (ms_fac * 1e-3) / 1e12 / fp64_sustained,
                     "dgemm_sustained_clocks": clk_dgemm.summary()},
        "roofline_solve": {"bound": "hbm", "achieved": B_solve / (ms_sol * 1e-3) / 1e9, "peak": hbm_peak,
                           "unit": "GB/s", "frac": B_solve / (ms_sol * 1e-3) / 1e9 / hbm_peak,
                           "traffic": traffic.get("solve_q1_bytes")},
        "e2e": {"value": F / (ms_e2e_fac * 1e-3) / 1e12, "unit": "TFLOP/s", "factor_ms": ms_e2e_fac,
                "solve_ms": ms_e2e_sol, "h2d_bytes_per_step": h2d + b1.nbytes, "d2h_bytes_per_step": u2.nbytes,
                "matches_device_run": same},
        "residual": resid,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "producer_s": t_prod,
        "diagnostics": {"max_z_cond": max_zc, "cholesky_fallbacks": n_fallbacks},
    }
    if cpu is not None:
        line["cpu_baseline"] = {"value": cpu["factor_tflops"], "unit": "TFLOP/s", "cores": cpu["cores"], "kind": "port",
                                "sample": cpu["sample"], "solve_ms_extrapolated": cpu["solve_ms_extrapolated"],
                                "solve_telescoping_ms_extrapolated": cpu["solve_telescoping_ms_extrapolated"]}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
