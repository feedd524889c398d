"""The library's batched fp64 DMMA GEMM (csrc/gemm.cuh, every product of the
factorization runs through it) against torch's fp64 matmul on the same inputs,
through the C-ABI test hook ks_test_gemm: each tile shape the dispatcher picks
(64x64, 128x64 with TMA staging, the N <= 64 panels), both operand orders, the
alpha/beta forms, and the triangular forms -- tri = 1 (tiles above the diagonal
skipped: the leaf Gaussian blocks) and tri = 2 (a symmetric product computed on
the tiles on and below the diagonal and mirrored by the epilogue: C = P_l H_l P_l^T
and the Schur update H = C - F S^-1 E, solver.py:154-164). Floating point:
tolerance 1e-13 relative to |A||B| (fp64 accumulation order differs from cuBLAS)."""
import ctypes as C

import pytest

pytestmark = pytest.mark.gpu


def _gemm(lib, A, B, Cm, alpha, beta, ta, tb, tri=0):
    import torch
    batch = A.shape[0]
    M, N = Cm.shape[1], Cm.shape[2]
    K = A.shape[1] if ta else A.shape[2]
    rc = lib.ks_test_gemm(M, N, K, batch, tri, C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()),
                          C.c_void_p(Cm.data_ptr()), A.stride(1), A.stride(0), B.stride(1), B.stride(0),
                          Cm.stride(1), Cm.stride(0), alpha, beta, int(ta), int(tb), None)
    assert rc == 0
    torch.cuda.synchronize()


@pytest.mark.parametrize("M,N,K,batch", [(256, 256, 256, 8), (512, 512, 512, 16), (320, 64, 192, 40),
                                         (1152, 64, 512, 128), (256, 32, 64, 8), (192, 16, 96, 8)])
@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False)])
def test_gemm_matches_torch(M, N, K, batch, ta, tb):
    import torch

    from paper_1602_01376_b200 import _lib
    lib = _lib.load()
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K + batch)
    A = torch.randn((batch, K, M) if ta else (batch, M, K), generator=g, device="cuda", dtype=torch.float64)
    B = torch.randn((batch, N, K) if tb else (batch, K, N), generator=g, device="cuda", dtype=torch.float64)
    C0 = torch.randn((batch, M, N), generator=g, device="cuda", dtype=torch.float64)
    opA = A.transpose(1, 2) if ta else A
    opB = B.transpose(1, 2) if tb else B
    for alpha, beta in [(1.0, 0.0), (-1.0, 1.0)]:
        Cm = C0.clone()
        _gemm(lib, A, B, Cm, alpha, beta, ta, tb)
        ref = alpha * torch.matmul(opA, opB) + beta * C0
        scale = float(torch.matmul(opA.abs(), opB.abs()).max())
        assert float((Cm - ref).abs().max()) <= 1e-13 * scale


@pytest.mark.parametrize("S,K,batch", [(256, 256, 8), (256, 1024, 16), (512, 512, 16), (512, 768, 32)])
def test_symmetric_forms(S, K, batch):
    """tri = 1 leaves the tiles strictly above the diagonal untouched; tri = 2 returns
    the full symmetric product from the tiles on and below it (64x64 tiles for the
    small cases, 128x64 for the K >= 512 ones with enough tiles)."""
    import torch

    from paper_1602_01376_b200 import _lib
    lib = _lib.load()
    g = torch.Generator(device="cuda").manual_seed(S + K + batch)
    A = torch.randn((batch, S, K), generator=g, device="cuda", dtype=torch.float64)
    ref = torch.matmul(A, A.transpose(1, 2))
    scale = float(torch.matmul(A.abs(), A.abs().transpose(1, 2)).max())
    # tri = 2, C = A A^T (op(B) = B^T with B = A), and the beta form on a symmetric C
    Cm = torch.full((batch, S, S), float("nan"), device="cuda", dtype=torch.float64)
    _gemm(lib, A, A, Cm, 1.0, 0.0, False, True, tri=2)
    assert float((Cm - ref).abs().max()) <= 1e-13 * scale
    assert torch.equal(Cm.tril(-128), Cm.transpose(1, 2).tril(-128))  # mirrored tiles are bitwise transposes
    C0 = ref.clone()
    _gemm(lib, A, A, C0, -0.5, 1.0, False, True, tri=2)
    assert float((C0 - 0.5 * ref).abs().max()) <= 1e-13 * scale
    # tri = 1: the lower triangle is the product, tiles strictly above the diagonal keep their content
    Cm = torch.full((batch, S, S), -7.0, device="cuda", dtype=torch.float64)
    _gemm(lib, A, A, Cm, 1.0, 0.0, False, True, tri=1)
    assert float((Cm.tril() - ref.tril()).abs().max()) <= 1e-13 * scale
    assert float(Cm[:, :64, S - 64:].min()) == -7.0 and float(Cm[:, :64, S - 64:].max()) == -7.0
