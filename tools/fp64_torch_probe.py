"""Library fp64 ceilings on the box (cuBLAS DGEMM, cuSOLVER batched potrf) for DESIGN.md."""
import time, torch
def t(f, reps=5):
    f(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); torch.cuda.synchronize(); best = min(best, a.elapsed_time(b))
    return best
for n in (1024, 4096, 8192):
    A = torch.randn(n, n, dtype=torch.float64, device="cuda"); B = torch.randn(n, n, dtype=torch.float64, device="cuda")
    ms = t(lambda: A @ B)
    print(f"DGEMM {n}^3: {2*n**3/ms/1e9:.2f} TFLOP/s")
for (bt, m) in ((64, 1024), (1024, 128), (128, 512)):
    A = torch.randn(bt, m, m, dtype=torch.float64, device="cuda"); A = A @ A.transpose(1, 2) + m * torch.eye(m, device="cuda", dtype=torch.float64)
    ms = t(lambda: torch.linalg.cholesky(A))
    print(f"cusolver batched potrf {bt}x{m}: {bt*m**3/3/ms/1e9:.3f} TFLOP/s ({ms:.2f} ms)")
    ms = t(lambda: torch.linalg.lu_factor(A))
    print(f"cusolver batched getrf {bt}x{m}: {bt*2*m**3/3/ms/1e9:.3f} TFLOP/s ({ms:.2f} ms)")
    bm = torch.bmm
    ms = t(lambda: bm(A, A))
    print(f"bmm {bt}x{m}: {bt*2*m**3/ms/1e9:.3f} TFLOP/s")
x = torch.empty(1 << 30, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
ms = t(lambda: y.copy_(x)); print(f"copy {2*8*(1<<30)/ms/1e6:.0f} GB/s")
