"""Does the DMMA GEMM rate depend on the operand data? Time the leaf SYRK on the
factor's real L21 rows, on the same rows with subnormals flushed, and on random data."""
import os, sys, ctypes as C
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_1602_01376_b200 as ks
from paper_1602_01376_b200 import _lib
from paper_1602_01376_b200.configs import CONFIGS
from producer import make_operator
cfg = CONFIGS["cfg3"]
op = make_operator(cfg)
hf = ks.factorize(op, cfg.lam)
lib = _lib.load()
M, S, R, nl = 1024, 256, 1280, 1024
base = lib.ks_debug_ptr(hf.handle, 5)
out = torch.empty(nl, S, S, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
def run(ptr, lda, sa):
    rc = lib.ks_test_gemm(S, S, M, nl, 0, C.c_void_p(ptr), C.c_void_p(ptr), C.c_void_p(out.data_ptr()), lda, sa, lda, sa, S, S * S, 1.0, 0.0, 0, 1, C.c_void_p(s))
    assert rc == 0
def t(f, reps=3):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [f() for _ in range(reps)]; e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
fl = 2.0 * S * S * M * nl
ms = t(lambda: run(base + M * M * 8, M, R * M)); print(f"real L21: {fl/ms/1e9:.2f} TF/s")
# copy L21 out
L21 = torch.empty(nl, S, M, dtype=torch.float64, device="cuda")
lib2 = torch.cuda
cp = torch.empty(0)
import numpy as np
# gather through a strided view: build from raw pointer via cudaMemcpy2D is not exposed; use ks_debug_copy per leaf is slow -> use torch from dlpack trick
# simpler: use cuda-python-free path: compute with ks_test_gemm alpha=1 copy (C = A * I)
eye = torch.eye(M, dtype=torch.float64, device="cuda").expand(nl, M, M).contiguous()
rc = lib.ks_test_gemm(S, M, M, nl, 0, C.c_void_p(base + M * M * 8), C.c_void_p(eye.data_ptr()), C.c_void_p(L21.data_ptr()), M, R * M, M, M * M, M, S * M, 1.0, 0.0, 0, 0, C.c_void_p(s))
assert rc == 0
del eye
torch.cuda.synchronize()
a = L21.abs()
tiny = ((a > 0) & (a < 2.2250738585072014e-308)).sum().item()
print("L21 subnormals:", tiny, "zeros:", (a == 0).sum().item(), "min nonzero:", a[a > 0].min().item(), "max:", a.max().item())
ms = t(lambda: run(L21.data_ptr(), M, S * M)); print(f"L21 copy: {fl/ms/1e9:.2f} TF/s")
L21f = torch.where(a < 1e-300, torch.zeros_like(L21), L21)
ms = t(lambda: run(L21f.data_ptr(), M, S * M)); print(f"L21 flushed (<1e-300 -> 0): {fl/ms/1e9:.2f} TF/s")
Rn = torch.randn_like(L21)
ms = t(lambda: run(Rn.data_ptr(), M, S * M)); print(f"random: {fl/ms/1e9:.2f} TF/s")
hb = lib.ks_debug_ptr(hf.handle, 6)
def run_h(ptr, lda, sa):
    rc = lib.ks_test_gemm(S, S, M, nl, 0, C.c_void_p(ptr), C.c_void_p(ptr), C.c_void_p(hb + 1023 * S * S * 8), lda, sa, lda, sa, S, S * S, 1.0, 0.0, 0, 1, C.c_void_p(s))
    assert rc == 0
ms = t(lambda: run_h(base + M * M * 8, M, R * M)); print(f"real L21 -> hbuf: {fl/ms/1e9:.2f} TF/s")
hf.refactorize(cfg.lam)
torch.cuda.synchronize()
ms = t(lambda: run(base + M * M * 8, M, R * M)); print(f"after refactorize, real L21 -> out: {fl/ms/1e9:.2f} TF/s")
ms = t(lambda: run_h(base + M * M * 8, M, R * M)); print(f"after refactorize, real L21 -> hbuf: {fl/ms/1e9:.2f} TF/s")
ln = lib.ks_debug_ptr(hf.handle, 7)
def run_idx(ptr, lda, sa):
    rc = lib.ks_test_gemm_cidx(S, S, M, nl, C.c_void_p(ptr), C.c_void_p(ptr), C.c_void_p(hb), C.c_void_p(ln), lda, sa, lda, sa, S, S * S, 0, 1, C.c_void_p(s))
    assert rc == 0
ms = t(lambda: run_idx(base + M * M * 8, M, R * M)); print(f"real L21 -> hbuf via node idx: {fl/ms/1e9:.2f} TF/s")
os.environ["KS_TRACE"] = "1"
torch.cuda.synchronize()
ts = []
for i in range(40):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); run_idx(base + M * M * 8, M, R * M); e1.record()
    ts.append((e0, e1))
torch.cuda.synchronize()
print("back-to-back SYRK ms:", [round(a.elapsed_time(b), 2) for a, b in ts])
# interleave with a factorization
for i in range(2):
    hf.refactorize(cfg.lam)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); run_idx(base + M * M * 8, M, R * M); e1.record(); torch.cuda.synchronize()
    print("SYRK right after a refactorize:", round(e0.elapsed_time(e1), 2), "ms")
