"""One factor+solve step at a config, bracketed by cudaProfilerStart/Stop for
`ncu --profile-from-start off` (the producer's torch kernels stay outside)."""
import argparse, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_1602_01376_b200 as ks
from paper_1602_01376_b200.configs import CONFIGS
from producer import make_operator, make_rhs

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--q", type=int, default=1)
ap.add_argument("--what", default="both", choices=["both", "factor", "solve"])
a = ap.parse_args()
cfg = CONFIGS[a.config]
op = make_operator(cfg)
hf = ks.factorize(ks.from_arrays(op), cfg.lam)
hf.set_profiling(True)
B = torch.from_numpy(make_rhs(cfg, op["perm"], a.q)).cuda()
ks.solve_many(hf, B)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
if a.what in ("both", "factor"):
    hf.refactorize(cfg.lam)
if a.what in ("both", "solve"):
    ks.solve_many(hf, B)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
if os.environ.get("KS_TRACE") == "1":
    hf.refactorize(cfg.lam)
    print(hf.trace_report())
    print("levels", [round(x, 3) for x in hf.level_ms()])
if os.environ.get("KS_TRACE") == "1":
    ks.solve_many(hf, B)
    torch.cuda.synchronize()
    print("solve trace q=%d" % a.q)
    print(hf.trace_report())
