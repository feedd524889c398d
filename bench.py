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

from paper_1602_01376_b200 import launch  # noqa: E402  (no torch / CUDA import)

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
# CPU baseline: the reference's own kernelsolve (installed unmodified into
# baseline/_ref) on a bounded sample of the workload; the
# oracle port (oracle/ks_oracle.py) only when the reference is not installed.
# ---------------------------------------------------------------------------
REF_DIR = os.path.join(ROOT, "baseline", "_ref")
SAMPLE = "cfg3s"  # the reference's own cfg3-shaped operator: N=4096, 4 leaves m=1024, 3 internal s=256, d=28
SAMPLE_DESC = ("cfg3-shaped reference operator (tests/golden/cfg3s.npz, reference compression output) N=4096: "
               "4 leaves m=1024 + 3 internal nodes s=256, d=28; factorize measured, the full-size recursive solve "
               "extrapolated x(1024/4)^2 leaf solves (solver.py:216-237 visits a level-l node 2^l times)")


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_installed() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "kernelsolve"))


def _reference_ck(ksr, g: dict):
    """The reference's CompressedKernel for a marshalled operator (compress.py:93-142):
    its own PointSet / PartitionTree / Skeleton types, leaf blocks and couplings
    evaluated by its own kernel_block (compress.py:271-283)."""
    n_nodes = g["node_begin"].size
    nodes = []
    for v in range(n_nodes):
        ch = None if g["node_left"][v] < 0 else (int(g["node_left"][v]), int(g["node_right"][v]))
        nodes.append(ksr.TreeNode(id=v, level=int(g["node_level"][v]), begin=int(g["node_begin"][v]),
                                  end=int(g["node_end"][v]), children=ch))
    depth = int(g["node_level"].max()) + 1
    pts = ksr.PointSet(np.asarray(g["coords"], dtype=np.float64))
    tree = ksr.PartitionTree(nodes=nodes, perm=np.asarray(g["perm"], dtype=np.int64),
                             leaf_size=int(max(nd.size for nd in nodes if nd.is_leaf)), depth=depth)
    spec = ksr.KernelSpec("gaussian", bandwidth=float(g["h"]))
    skels, leaf_diag, couplings = [None] * n_nodes, {}, {}
    for v in range(n_nodes):
        r = int(g["rank"][v])
        if r:
            sk = g["skel"][g["skel_off"][v]:g["skel_off"][v + 1]]
            coeff = g["coeff"][g["coeff_off"][v]:g["coeff_off"][v + 1]].reshape(r, -1)
            nd = nodes[v]
            cand = (tree.node_points(v) if nd.is_leaf else None)
            skels[v] = ksr.Skeleton(node_id=v, cand=cand, skel=np.asarray(sk, np.int64), coeff=coeff)
    for v in range(n_nodes):
        nd = nodes[v]
        if nd.is_leaf:
            ids = tree.node_points(v)
            leaf_diag[v] = ksr.kernel_block(spec, pts, ids, ids)
        else:
            l, r = nd.children
            skels_v = skels[v]
            if skels_v is not None:
                skels_v.cand = np.concatenate([skels[l].skel, skels[r].skel])
            couplings[v] = ksr.kernel_block(spec, pts, skels[l].skel, skels[r].skel)
    params = ksr.CompressParams(tol=1e-5, max_rank=int(g["rank"].max()), seed=0)
    return ksr.CompressedKernel(points=pts, tree=tree, spec=spec, params=params, skeletons=skels,
                                leaf_diag=leaf_diag, couplings=couplings, neighbors=None)


def ref_worker(setting: str, steps: int, warmup: int) -> None:
    """One CPU-baseline setting, run in its own process so the BLAS thread
    count is fixed before numpy loads: "i" = threads=1 with
    BLAS on all cores (the CLI default, report.py:125), "ii" = threads=ncores
    with BLAS single-threaded. Prints one JSON object of per-step times."""
    sys.path.insert(0, REF_DIR)
    import kernelsolve as ksr  # the unmodified reference (baseline/_ref)

    from paper_1602_01376_b200 import yardstick

    with np.load(os.path.join(ROOT, "tests", "golden", f"{SAMPLE}.npz")) as z:
        g = {k: z[k] for k in z.files}
    ck = _reference_ck(ksr, g)
    lam = float(g["lam"])
    b = g["b"][:, :1]
    threads = 1 if setting == "i" else (os.cpu_count() or 1)
    tf, ts = [], []
    for it in range(warmup + steps):
        t0 = time.perf_counter()
        hf = ksr.factorize(ck, lam, threads=threads)
        t1 = time.perf_counter()
        u = ksr.solve_many(hf, b)
        t2 = time.perf_counter()
        if it >= warmup:
            tf.append(t1 - t0)
            ts.append(t2 - t1)
    err = float(np.linalg.norm(u - g["u"][:, :1]) / np.linalg.norm(g["u"][:, :1]))
    print(json.dumps({"setting": setting, "threads": threads, "blas_threads": os.environ.get("OPENBLAS_NUM_THREADS"),
                      "factor_s": tf, "solve_s": ts, "flops": yardstick.factor_flops(g), "u_vs_golden": err}),
          flush=True)


def reference_cpu(steps: int, warmup: int) -> dict:
    """Both thread settings of the reference on the host; the better one."""
    ncores = os.cpu_count() or 1
    runs = []
    for setting, blas in (("i", str(ncores)), ("ii", "1")):
        env = dict(os.environ)
        for k in ("RANK", "LOCAL_RANK", "WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT"):
            env.pop(k, None)
        env.update(OPENBLAS_NUM_THREADS=blas, OMP_NUM_THREADS=blas, MKL_NUM_THREADS=blas, CUDA_VISIBLE_DEVICES="")
        out = subprocess.run([sys.executable, os.path.abspath(__file__), "--ref-worker", setting, "--steps", str(steps),
                              "--warmup", str(warmup)], env=env, capture_output=True, text=True, timeout=1800)
        if out.returncode != 0:
            raise RuntimeError(f"reference worker {setting} failed: {out.stderr[-2000:]}")
        runs.append(json.loads(out.stdout.strip().splitlines()[-1]))
    for r in runs:
        r["factor_tflops"] = r["flops"] / float(np.median(r["factor_s"])) / 1e12
    best = max(runs, key=lambda r: r["factor_tflops"])
    leaves_sample, leaves_full = 4, 1024
    return {
        "factor_tflops": best["factor_tflops"],
        "factor_s_sample": float(np.median(best["factor_s"])),
        "solve_ms_extrapolated": float(np.median(best["solve_s"])) * (leaves_full / leaves_sample) ** 2 * 1e3,
        "cores": best["threads"] if best["setting"] == "ii" else ncores,
        "kind": "reference",
        "setting": ("threads=1, OpenBLAS on %d cores" % ncores) if best["setting"] == "i"
        else ("threads=%d, OPENBLAS_NUM_THREADS=1" % best["threads"]),
        "settings": {r["setting"]: {"factor_tflops": r["factor_tflops"], "threads": r["threads"],
                                    "OPENBLAS_NUM_THREADS": r["blas_threads"],
                                    "factor_s": r["factor_s"], "solve_s": r["solve_s"]} for r in runs},
        "u_vs_golden": best["u_vs_golden"],
        "cpu_model": cpu_model(),
        "sample": SAMPLE_DESC,
    }


def cpu_sample(repeats: int = 1) -> dict:
    """Fallback when the reference is not installed: the oracle port of the
    reference algorithm (oracle/ks_oracle.py, numpy + the box's BLAS threads)
    on the same sample."""
    from oracle import ks_oracle as O
    from paper_1602_01376_b200 import yardstick

    with np.load(os.path.join(ROOT, "tests", "golden", f"{SAMPLE}.npz")) as z:
        g = {k: z[k] for k in z.files}
    prob = O.Problem(g)
    lam = float(g["lam"])
    b = g["b"][:, :1]
    tf, ts = [], []
    for _ in range(repeats):
        t0 = time.perf_counter()
        of = O.factorize(prob, lam)
        t1 = time.perf_counter()
        O.solve_many_recursive(of, b)
        t2 = time.perf_counter()
        tf.append(t1 - t0)
        ts.append(t2 - t1)
    F = yardstick.factor_flops(g)
    return {
        "factor_tflops": F / float(np.median(tf)) / 1e12,
        "factor_s_sample": float(np.median(tf)),
        "solve_ms_extrapolated": float(np.median(ts)) * (1024 / 4) ** 2 * 1e3,
        "cores": os.cpu_count(), "kind": "port", "cpu_model": cpu_model(),
        "setting": "OPENBLAS_NUM_THREADS=%s" % os.environ.get("OPENBLAS_NUM_THREADS", "default"),
        "sample": SAMPLE_DESC.replace("reference operator", "reference operator, oracle port"),
    }


def cpu_baseline(steps: int = 1, warmup: int = 1) -> dict:
    return reference_cpu(steps, warmup) if reference_installed() else cpu_sample(steps)


def cpu_line(cb: dict) -> dict:
    return {"value": cb["factor_tflops"], "unit": "TFLOP/s", "cores": cb["cores"], "kind": cb["kind"],
            "sample": cb["sample"], "setting": cb["setting"], "cpu_model": cb["cpu_model"],
            "solve_ms_extrapolated": cb["solve_ms_extrapolated"], "settings": cb.get("settings")}


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    t0 = time.perf_counter()
    cb = cpu_baseline(args.steps, args.warmup)
    wall = time.perf_counter() - t0
    val = cb["factor_tflops"]
    line = {
        "metric": METRIC, "value": val, "unit": "TFLOP/s", "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["factor_s_sample"] * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg3 factor+solve q=1, bounded CPU sample (N=4096 at cfg3's leaf/rank/d shape)",
                   "n": 1048576, "d": 28, "leaf": 1024, "rank": 256, "h": 1.5, "lambda": 0.1, "q": 1,
                   "sample_n": 4096},
        "solve_ms": cb["solve_ms_extrapolated"],
        "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": cb["cores"], "kind": cb["kind"],
                         "sample": cb["sample"], "setting": cb["setting"], "cpu_model": cb["cpu_model"],
                         "settings": cb.get("settings")},
        "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": wall,
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
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or args.sharded:
        return run_multi(args)
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
    cpu = cpu_baseline() if not args.no_cpu else None
    B_solve = yardstick.solve_bytes(op, 1)
    # DRAM bytes per factorization / per q=1 solve from the committed ncu capture
    # (profiles/r02_dram_traffic.json: cold caches, an upper bound), config 3 only
    traffic = {}
    tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r02_dram_traffic.json")
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
        line["cpu_baseline"] = cpu_line(cpu)
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# N GPUs: subtree sharding, one process per GPU over NCCL
# ---------------------------------------------------------------------------
def _broadcast_operator(torch, dist, op: dict | None, rank: int) -> dict:
    """Rank 0's operator arrays to every rank (NCCL broadcast of device copies):
    every shard factors bit-identical inputs."""
    meta = [None]
    if rank == 0:
        meta[0] = {k: (np.asarray(v).shape, str(np.asarray(v).dtype)) for k, v in op.items()}
    dist.broadcast_object_list(meta, src=0)
    out = {}
    for k, (shape, dt) in meta[0].items():
        if rank == 0:
            a = np.ascontiguousarray(np.asarray(op[k]))
            t = torch.from_numpy(a.reshape(-1) if a.ndim else a.reshape(1)).cuda()
        else:
            t = torch.empty(int(np.prod(shape)) if len(shape) else 1, dtype=getattr(torch, dt), device="cuda")
        dist.broadcast(t, src=0)
        a = t.cpu().numpy()
        out[k] = a.reshape(shape) if len(shape) else a.reshape(())
        del t
    return out


def _nccl_summary() -> dict:
    """Which NCCL transports the run used (NCCL_DEBUG=INFO lines, NCCL_DEBUG_FILE)."""
    import glob

    pat = os.environ.get("NCCL_DEBUG_FILE", "")
    files = glob.glob(pat.replace("%h", "*").replace("%p", "*")) if pat else []
    text = ""
    for fn in files:
        try:
            with open(fn, errors="replace") as fh:
                text += fh.read()
        except OSError:
            pass
    return {"debug": os.environ.get("NCCL_DEBUG"), "log_files": len(files),
            "nvls": ("NVLS" in text) and ("NVLS multicast support is not available" not in text),
            "p2p_nvlink": ("P2P/CUMEM" in text) or ("via P2P" in text) or ("NVLink" in text),
            "lines": len(text.splitlines())}


def run_multi(args) -> None:
    import torch
    import torch.distributed as dist

    import paper_1602_01376_b200 as ks
    from paper_1602_01376_b200 import distributed as kd
    from paper_1602_01376_b200 import yardstick
    from paper_1602_01376_b200.configs import CONFIGS

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if torch.cuda.device_count() <= local:
        raise SystemExit(f"rank {rank}: LOCAL_RANK {local} but only {torch.cuda.device_count()} visible GPU(s)")
    torch.cuda.set_device(local)
    # the transport NCCL picks (NVLS, P2P over NVLink) goes to a log file, summarized in the JSON line
    if os.environ.get("NCCL_DEBUG", "").upper() not in ("INFO", "TRACE"):
        os.environ["NCCL_DEBUG"] = "INFO"
    os.environ.setdefault("NCCL_DEBUG_FILE", "/tmp/ks_nccl.%h.%p.log")
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = CONFIGS[args.config]
    op = None
    t0 = time.perf_counter()
    if rank == 0:
        from producer import make_operator
        op = make_operator(cfg, device="cuda", verbose=args.verbose)
    op = _broadcast_operator(torch, dist, op, rank)
    t_prod = time.perf_counter() - t0
    from producer import make_rhs

    prob = ks.from_arrays(op)
    root, peers = kd.shard_for(prob, world, rank)
    F = yardstick.factor_flops(op)
    B_solve = yardstick.solve_bytes(op, 1)
    b_np = make_rhs(cfg, op["perm"], 1)
    b = torch.from_numpy(b_np).cuda()
    fp64_peak = measure_fp64_peak(torch)
    stream = torch.cuda.current_stream()
    sh = kd.LibShard(prob, root, local)
    for _ in range(args.warmup):
        kd.factorize_sharded(sh, cfg.lam)
        kd.solve_many_sharded(sh, b, gather=False)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    launches = 0
    dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        for i in range(args.steps):
            ev[i][0].record(stream)
            kd.factorize_sharded(sh, cfg.lam)
            ev[i][1].record(stream)
            kd.solve_many_sharded(sh, b, gather=False)
            ev[i][2].record(stream)
            launches += sh.lib.ks_last_launches(sh.h, 0) + sh.lib.ks_last_launches(sh.h, 1)
        torch.cuda.synchronize()
        dist.barrier()
    tf = float(np.mean([e[0].elapsed_time(e[1]) for e in ev]))
    ts = float(np.mean([e[1].elapsed_time(e[2]) for e in ev]))
    t = torch.tensor([tf, ts, fp64_peak, float(launches)], dtype=torch.float64, device="cuda")
    tmax = t.clone()
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    tsum = t.clone()
    dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
    tf, ts = float(tmax[0]), float(tmax[1])
    peak_job, launches_job = float(tsum[2]), int(tsum[3])
    clocks = [None] * world
    dist.all_gather_object(clocks, clk.summary())
    # p = N agrees with p = 1: the gathered sharded solution vs an unsharded factor on rank 0
    X = kd.solve_many_sharded(sh, b, gather=True)
    dev_bytes = sh.lib.ks_device_bytes(sh.h)
    sh.close()
    agree = None
    if rank == 0:
        hf1 = ks.factorize(prob, cfg.lam)
        X1 = ks.solve_many(hf1, b)
        agree = float(torch.linalg.norm(X - X1) / torch.linalg.norm(X1))
        Ku = ks.hss_matvec(hf1, X)
        resid = float(torch.linalg.norm(Ku + cfg.lam * X - b) / torch.linalg.norm(b))
        hf1.close()
        del X1, Ku
    del X
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    # e2e through the public API from pinned host buffers: every rank creates its
    # shard from the host operator (uploads its subtree's inputs), the sharded
    # factorization and solve, and rank 0 reads the gathered solution back
    pin, _ = _pinned_problem(torch, op)
    pin_prob = ks.from_arrays(pin)
    b_pin = torch.from_numpy(b_np).pin_memory()
    e2e_f, e2e_s, up_bytes = [], [], 0
    for i in range(3):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sf = kd.factorize_distributed(pin_prob, cfg.lam)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        Xh = sf.solve_many(b_pin, gather=True)
        if rank == 0:
            Xh.cpu().numpy()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        up_bytes = sf.backend.lib.ks_upload_bytes(sf.backend.h)
        sf.close()
        tt = torch.tensor([t1 - t0, t2 - t1], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_f.append(float(tt[0]))
        e2e_s.append(float(tt[1]))
    ub = torch.tensor([float(up_bytes)], dtype=torch.float64, device="cuda")
    dist.all_reduce(ub, op=dist.ReduceOp.SUM)
    h2d_job = int(ub.item()) + int(b_np.nbytes)  # each rank copies its operator part; B's rows once in total
    ms_e2e_f, ms_e2e_s = float(np.median(e2e_f)) * 1e3, float(np.median(e2e_s)) * 1e3
    cpu = cpu_baseline() if (rank == 0 and not args.no_cpu) else None
    nccl = _nccl_summary() if rank == 0 else None
    dist.barrier()
    if rank == 0:
        val = F / (tf * 1e-3) / 1e12
        line = {
            "metric": METRIC, "value": val, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tf + ts, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (config recipe points from the reference RNG; tree restated bit-exactly; "
                    "skeletons/P by the GPU producer on rank 0, broadcast to every rank)",
            "config": {"workload": f"{cfg.name} factor+solve q=1, subtree-sharded over {world} GPUs", "n": cfg.n,
                       "d": cfg.d, "leaf": cfg.leaf_size, "rank": cfg.max_rank, "h": cfg.h, "lambda": cfg.lam,
                       "q": 1, "parallelism": f"subtree{world} (NCCL all-gather of skeleton blocks)",
                       "l2": "inputs larger than L2 (%.1f GB per GPU)" % (dev_bytes / 1e9)},
            "factor_ms": tf, "solve_ms": ts,
            "roofline": {"bound": "tensor", "achieved": val, "peak": peak_job, "unit": "TFLOP/s",
                         "frac": val / peak_job, "traffic": None,
                         "kernel": f"whole factorization over {world} GPUs; peak = sum of the ranks' live cuBLAS DGEMM"},
            "roofline_solve": {"bound": "hbm", "achieved": B_solve / (ts * 1e-3) / 1e9,
                               "peak": world * float(_peaks().get("hbm_gbs", 6538.9)), "unit": "GB/s",
                               "frac": B_solve / (ts * 1e-3) / 1e9 / (world * float(_peaks().get("hbm_gbs", 6538.9)))},
            "e2e": {"value": F / (ms_e2e_f * 1e-3) / 1e12, "unit": "TFLOP/s", "factor_ms": ms_e2e_f,
                    "solve_ms": ms_e2e_s, "h2d_bytes_per_step": h2d_job, "d2h_bytes_per_step": int(b_np.nbytes)},
            "p1_vs_pN_rel": agree, "residual": resid,
            "gpu_launches": launches_job,
            "clocks": clocks[0], "clocks_per_rank": clocks,
            "nccl": nccl, "producer_s": t_prod,
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu_line(cpu)
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--ref-worker", default=None, help=argparse.SUPPRESS)
    # the sharded (multi-GPU) code path on a single rank (under torchrun with 1 process): a check of
    # run_multi where only one GPU is available
    ap.add_argument("--sharded", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.ref_worker:
        ref_worker(args.ref_worker, args.steps, args.warmup)
        return
    if args.gpus > 1 and not launch.under_launcher():
        # one process per GPU: start the ranks ourselves (the driver may also
        # launch this script under torchrun, which lands in run_multi directly)
        env = {"NCCL_DEBUG": os.environ.get("NCCL_DEBUG", "INFO"),
               "NCCL_DEBUG_FILE": os.environ.get("NCCL_DEBUG_FILE", "/tmp/ks_nccl.%h.%p.log")}
        r = launch.spawn(args.gpus, os.path.abspath(__file__), sys.argv[1:], env=env)
        raise SystemExit(r.returncode)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
