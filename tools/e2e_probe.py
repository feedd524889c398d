"""Break the end-to-end (host-buffer) factor/solve time into its pieces:
ks_create (validation + uploads + allocation), the first (eager) ks_factorize,
ks_solve with host buffers, ks_destroy. Usage: python tools/e2e_probe.py [--config 3]"""

import argparse
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1602_01376_b200 as ks  # noqa: E402
from paper_1602_01376_b200 import _lib  # noqa: E402
from paper_1602_01376_b200.configs import CONFIGS  # noqa: E402
from producer import make_operator, make_rhs  # noqa: E402
from bench import _pinned_problem  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    op = make_operator(cfg, device="cuda")
    torch.cuda.empty_cache()  # the producer's cached blocks would crowd the library's pool
    pin, h2d = _pinned_problem(torch, op)
    prob = ks.from_arrays(pin)
    b = torch.from_numpy(make_rhs(cfg, op["perm"], 1)).pin_memory().numpy()
    x = torch.empty(b.shape, dtype=torch.float64).pin_memory().numpy()
    lib = _lib.load()
    cp = prob.to_c()
    print(f"h2d bytes {h2d / 1e9:.3f} GB")
    for r in range(a.reps):
        h = C.c_void_p()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rc = lib.ks_create(C.byref(cp), 0, C.byref(h))
        assert rc == 0, _lib.last_error()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        assert lib.ks_factorize(h, cfg.lam, None) == 0
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        assert lib.ks_solve(h, b.ctypes.data, x.ctypes.data, 1, None) == 0
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        assert lib.ks_solve(h, b.ctypes.data, x.ctypes.data, 1, None) == 0
        torch.cuda.synchronize()
        t4 = time.perf_counter()
        lib.ks_destroy(h)
        torch.cuda.synchronize()
        t5 = time.perf_counter()
        ms = lambda u, v: (v - u) * 1e3  # noqa: E731
        print(f"rep {r}: create {ms(t0, t1):.1f}  factorize {ms(t1, t2):.1f}  solve#1 {ms(t2, t3):.1f}  "
              f"solve#2 {ms(t3, t4):.1f}  destroy {ms(t4, t5):.1f} ms", flush=True)
    # the public API path as bench.py times it
    for r in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        hf = ks.factorize(prob, cfg.lam)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        ks.solve_many(hf, b)
        t2 = time.perf_counter()
        hf.close()
        print(f"api {r}: factorize {(t1 - t0) * 1e3:.1f}  solve_many {(t2 - t1) * 1e3:.1f} ms", flush=True)


if __name__ == "__main__":
    main()
