"""Our batched DMMA GEMM vs cuBLAS (torch.bmm) on the factorization's shapes."""
import os, sys, ctypes as C
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
from paper_1602_01376_b200 import _lib
lib = _lib.load()
lib.ks_test_gemm.restype = C.c_int
lib.ks_test_gemm.argtypes = [C.c_int]*5 + [C.c_void_p]*3 + [C.c_int64]*6 + [C.c_double, C.c_double, C.c_int, C.c_int, C.c_void_p]
def ours(M, N, K, batch, ta, tb, A, B, Cm, reps=5):
    s = torch.cuda.current_stream().cuda_stream
    def run():
        rc = lib.ks_test_gemm(M, N, K, batch, 0, A.data_ptr(), B.data_ptr(), Cm.data_ptr(),
                              A.stride(-2), A.stride(0), B.stride(-2), B.stride(0), Cm.stride(-2), Cm.stride(0),
                              1.0, 0.0, ta, tb, C.c_void_p(s))
        assert rc == 0, rc
    run(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [run() for _ in range(reps)]; e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
def ref(f, reps=5):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [f() for _ in range(reps)]; e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for (M, N, K, batch) in [(256, 256, 1024, 1024), (1280, 64, 512, 1024), (768, 64, 64, 1024), (512, 512, 512, 128), (256, 256, 256, 512), (736, 256, 256, 512)]:
    A = torch.randn(batch, M, K, dtype=torch.float64, device="cuda")
    B = torch.randn(batch, N, K, dtype=torch.float64, device="cuda")
    Cm = torch.empty(batch, M, N, dtype=torch.float64, device="cuda")
    t = ours(M, N, K, batch, 0, 1, A, B, Cm)
    err = (Cm - torch.bmm(A, B.transpose(1, 2))).abs().max().item()
    tr = ref(lambda: torch.bmm(A, B.transpose(1, 2), out=Cm))
    fl = 2.0 * M * N * K * batch
    print(f"NT {M}x{N}x{K} x{batch}: ours {fl/t/1e9:6.2f} TF/s  cublas {fl/tr/1e9:6.2f} TF/s  maxerr {err:.1e}", flush=True)
    del A, B, Cm
# the leaf SYRK exactly as the factorization issues it: A = L21 rows inside the
# (m+s) x m leaf trapezoid (batch stride (m+s)*m), C = H buffer indexed by node id
R, M, S, nl = 1280, 1024, 256, 1024
big = torch.randn(nl, R, M, dtype=torch.float64, device="cuda")
A = big[:, M:, :]
Hb = torch.empty(2 * nl, S, S, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
def run_syrk():
    rc = lib.ks_test_gemm(S, S, M, nl, 0, A.data_ptr(), A.data_ptr(), Hb.data_ptr() + nl * S * S * 8 - 0,
                          M, R * M, M, R * M, S, S * S, 1.0, 0.0, 0, 1, C.c_void_p(s))
    assert rc == 0
t = ref(run_syrk)
print(f"leaf SYRK layout 256x256x1024 x1024: ours {2.0*S*S*M*nl/t/1e9:6.2f} TF/s")
A2 = A.contiguous()
def run2():
    rc = lib.ks_test_gemm(S, S, M, nl, 0, A2.data_ptr(), A2.data_ptr(), Hb.data_ptr(), M, S * M, M, S * M, S, S * S,
                          1.0, 0.0, 0, 1, C.c_void_p(s))
    assert rc == 0
t = ref(run2)
print(f"same, contiguous A: ours {2.0*S*S*M*nl/t/1e9:6.2f} TF/s")
