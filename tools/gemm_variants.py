import os, sys, ctypes as C, subprocess
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
if len(sys.argv) == 1:
    for v in range(6):
        out = subprocess.run([sys.executable, __file__, str(v)], env={**os.environ, "KS_GEMM_VARIANT": str(v)}, capture_output=True, text=True)
        print(f"variant {v}: {out.stdout.strip()} {out.stderr.strip()[-200:]}", flush=True)
    sys.exit()
import torch
from paper_1602_01376_b200 import _lib
lib = _lib.load()
s = torch.cuda.current_stream().cuda_stream
def t(f, reps=3):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [f() for _ in range(reps)]; e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
res = []
for (M, N, K, batch, ta, tb) in [(1280, 64, 512, 1024, 0, 1), (256, 256, 1024, 1024, 0, 1), (736, 256, 256, 512, 0, 0), (1216, 64, 64, 1024, 0, 1)]:
    A = torch.randn(batch, K if ta else M, M if ta else K, dtype=torch.float64, device="cuda")
    B = torch.randn(batch, N if tb else K, K if tb else N, dtype=torch.float64, device="cuda")
    Cm = torch.empty(batch, M, N, dtype=torch.float64, device="cuda")
    def run():
        rc = lib.ks_test_gemm(M, N, K, batch, 0, A.data_ptr(), B.data_ptr(), Cm.data_ptr(), A.stride(-2), A.stride(0), B.stride(-2), B.stride(0), Cm.stride(-2), Cm.stride(0), 1.0, 0.0, ta, tb, C.c_void_p(s))
        assert rc == 0, rc
    ms = t(run)
    res.append(f"{M}x{N}x{K}:{2.0*M*N*K*batch/ms/1e9:.1f}")
    del A, B, Cm
print(" ".join(res))
