"""Concurrent solves on one factor (the reference's contract: a HierFactor is
immutable and shared, solves on it are safe, solver.py:77-89, SPEC concurrency
model). Every ks_solve runs in a workspace of its own, so solves from several
host threads and on several CUDA streams give bit-identical results to the
same solves run one at a time."""
import threading

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg2(golden):
    import paper_1602_01376_b200 as ks
    g = golden("cfg2s")
    hf = ks.factorize(g, float(g["lam"]))
    yield g, hf
    hf.close()


def _rhs(n, k, q):
    return np.random.default_rng(100 + k).standard_normal((n, q))


def test_threads_host_buffers(cfg2):
    import paper_1602_01376_b200 as ks
    g, hf = cfg2
    n = hf.n
    qs = [1, 3, 8, 1, 16, 2, 1, 32]
    B = [_rhs(n, k, q) for k, q in enumerate(qs)]
    ref = [ks.solve_many(hf, b) for b in B]
    out = [None] * len(B)
    errs = []

    def work(k):
        try:
            for _ in range(3):
                out[k] = ks.solve_many(hf, B[k])
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=work, args=(k,)) for k in range(len(B))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for k in range(len(B)):
        assert np.array_equal(out[k], ref[k]), (k, rel(out[k], ref[k]))


def test_streams_device_buffers(cfg2):
    import torch

    import paper_1602_01376_b200 as ks
    g, hf = cfg2
    n = hf.n
    B = [torch.from_numpy(_rhs(n, 50 + k, q)).cuda() for k, q in enumerate([1, 2, 8, 1])]
    ref = [ks.solve_many(hf, b.cpu().numpy()) for b in B]
    streams = [torch.cuda.Stream() for _ in B]
    outs = [None] * len(B)
    torch.cuda.synchronize()
    for _ in range(4):  # issue all solves before any completes: they overlap on the device
        for k, (b, s) in enumerate(zip(B, streams)):
            with torch.cuda.stream(s):
                outs[k] = ks.solve_many(hf, b)
    torch.cuda.synchronize()
    for k in range(len(B)):
        assert np.array_equal(outs[k].cpu().numpy(), ref[k]), k
    # matvec concurrently with solves
    with torch.cuda.stream(streams[0]):
        y = ks.hss_matvec(hf, B[1])
    with torch.cuda.stream(streams[1]):
        x = ks.solve_many(hf, B[1])
    torch.cuda.synchronize()
    assert np.array_equal(x.cpu().numpy(), ref[1])
    assert np.array_equal(y.cpu().numpy(), ks.hss_matvec(hf, B[1].cpu().numpy()))
