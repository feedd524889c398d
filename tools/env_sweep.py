"""Factorization time (graph mode, device-resident) for several values of one
environment knob read at enqueue time, e.g.
  python tools/env_sweep.py KS_HAGER_CTAS 32 64 96 148"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1602_01376_b200 as ks  # noqa: E402
from paper_1602_01376_b200.configs import CONFIGS  # noqa: E402
from producer import make_operator  # noqa: E402

name, values = sys.argv[1], sys.argv[2:]
cfg = CONFIGS[os.environ.get("CFG", "cfg3")]
prob = ks.from_arrays(make_operator(cfg, device="cuda"))
st = torch.cuda.current_stream()
for v in values:
    os.environ[name] = v
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
    print(f"{name}={v}: factor {np.mean(ts):.2f} ms (min {np.min(ts):.2f})", flush=True)
    hf.close()
