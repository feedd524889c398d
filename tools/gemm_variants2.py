"""Tile-shape variants (KS_GEMM_VARIANT, read once per process) on the node
assembly shape: batched 256 x 256 x 256, NN and NT. Run once per variant."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_1602_01376_b200 import _lib  # noqa: E402

lib = _lib.load()
s = torch.cuda.current_stream().cuda_stream
for (M, N, K, batch) in [(256, 256, 256, 512), (256, 256, 256, 64), (256, 256, 256, 8), (512, 512, 512, 512)]:
    for tb in (0, 1):
        A = torch.randn(batch, M, K, dtype=torch.float64, device="cuda")
        B = torch.randn(batch, N, K, dtype=torch.float64, device="cuda") if tb else torch.randn(batch, K, N, dtype=torch.float64, device="cuda")
        Cm = torch.empty(batch, M, N, dtype=torch.float64, device="cuda")

        def run():
            rc = lib.ks_test_gemm(M, N, K, batch, 0, A.data_ptr(), B.data_ptr(), Cm.data_ptr(), A.stride(-2), A.stride(0),
                                  B.stride(-2), B.stride(0), Cm.stride(-2), Cm.stride(0), 1.0, 0.0, 0, tb, C.c_void_p(s))
            assert rc == 0
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            run()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 10
        print(f"v{os.environ.get('KS_GEMM_VARIANT', '0')} {'NT' if tb else 'NN'} {M}x{N}x{K} x{batch}: {2.0 * M * N * K * batch / t / 1e9:6.2f} TF/s", flush=True)
