"""Timeline of the persistent per-node LU at the root level (KS_SLAB_TRACE=1):
per step, the owner's panel phases and the look-ahead slab's phases (us from the
first stamp, %globaltimer)."""
import ctypes as C, os, sys
os.environ["KS_SLAB_TRACE"] = "1"
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import paper_1602_01376_b200 as ks
from paper_1602_01376_b200.configs import CONFIGS
from producer import make_operator

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
op = make_operator(cfg)
hf = ks.factorize(ks.from_arrays(op), cfg.lam)
hf.refactorize(cfg.lam)
lib = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_1602_01376_b200", "libinvaskit.so"))
n = 128 * 64 * 4
buf = (C.c_longlong * n)()
lib.ks_slab_trace(buf, n)
a = np.frombuffer(buf, dtype=np.int64).reshape(128, 64, 4).astype(np.float64)
t0 = a[a > 0].min()
a = np.where(a > 0, (a - t0) / 1e3, np.nan)
W = 32
T = 3 * 256 if cfg.name == "cfg3" else None
G = int(np.sum(~np.isnan(a[:, 0, 0])))
nst = int(np.sum(~np.isnan(a[np.arange(64) % 128, np.arange(64), 0]))) if False else None
print("slabs with stamps:", G)
hv = 1 if os.environ.get("KS_SLAB_PW") == "32" or os.environ.get("KS_SLAB_W") == "16" else 2
for j in range(64):
    o = j // hv
    own = a[o, j]
    if np.isnan(own[0]):
        break
    la = a[o + 1, j]
    last_upd = np.nanmax(a[:, j, 3])
    print(f"step {j:2d} owner: start {own[0]:8.1f} cols {own[1]-own[0]:6.1f} aug {own[2]-own[1]:6.1f} pub {own[3]-own[2]:6.1f} | "
          f"lookahead: acq +{la[0]-own[3]:5.1f} moves {la[1]-la[0]:5.1f} u12 {la[2]-la[1]:5.1f} upd {la[3]-la[2]:6.1f} | last update done {last_upd - own[3]:6.1f}")
