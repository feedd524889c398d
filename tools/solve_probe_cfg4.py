import os, sys, time
sys.path.insert(0, '/root/repo')
import torch, numpy as np
import paper_1602_01376_b200 as ks
from paper_1602_01376_b200.configs import CONFIGS
from producer import make_operator, make_rhs
cfg = CONFIGS['cfg4']
op = make_operator(cfg, device='cuda')
hf = ks.factorize(ks.from_arrays(op), cfg.lam)
print('diag', hf.diagnostics['cholesky_fallbacks'], len(hf.diagnostics['fallback_nodes']))
B = torch.from_numpy(make_rhs(cfg, op['perm'], 1)).cuda()
st = torch.cuda.current_stream()
for it in range(3):
    hf.refactorize(cfg.lam, st.cuda_stream)
    for j in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); X = ks.solve_many(hf, B); e1.record(st); torch.cuda.synchronize()
        print(it, j, 'solve ms', round(e0.elapsed_time(e1), 3))
