"""Timing-only ablation of the factorization schedule: KS_ABLATE is a bit mask of
pieces to skip (1 potrf64, 2 leaf diagonal update, 4 leaf update+TRSM GEMM,
8 leaf Gaussian GEMM, 16 leaf SYRK, 32 coupling/aug init, 64 node assembly GEMMs,
128 LU of S + Schur, 256 condition estimates, 1024 all internal levels). The factors
are garbage; only the time says how much of the step each piece accounts for with
everything else overlapped as in the real schedule.
    python tools/ablate.py 0 1 2 4 8 16 ...      (CFG=cfg3 default)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1602_01376_b200 as ks  # noqa: E402
from paper_1602_01376_b200.configs import CONFIGS  # noqa: E402
from producer import make_operator  # noqa: E402

values = sys.argv[1:] or ["0"]
cfg = CONFIGS[os.environ.get("CFG", "cfg3")]
prob = ks.from_arrays(make_operator(cfg, device="cuda"))
st = torch.cuda.current_stream()
os.environ["KS_ABLATE"] = "0"
hf = ks.factorize(prob, cfg.lam)  # a real factorization first: buffers hold finite data
hf.close()
for v in values:
    os.environ["KS_ABLATE"] = v
    hf = ks.factorize(prob, cfg.lam)
    for _ in range(3):
        hf.refactorize(cfg.lam, st.cuda_stream)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        hf.refactorize(cfg.lam, st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"KS_ABLATE={v}: factor {np.mean(ts):.2f} ms (min {np.min(ts):.2f})", flush=True)
    hf.close()
