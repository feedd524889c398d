"""Reference compression output at N = 16384 (config 3 recipe: d = 28, leaf
1024, rank 256, h = 1.5), integer parts only, for the producer's bit-exactness
test (tests/test_producer.py): the tree permutation, ranks and skeleton ids
kernelsolve.build_tree + kernelsolve.compress produce (compress.py:145-287,
tree.py:84-172). Run in the build container (needs /root/reference):

    python tests/golden/make_producer_golden.py
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import kernelsolve as ks  # noqa: E402  (reference, build container only)

from make_golden import _cfg, build, marshal  # noqa: E402

if __name__ == "__main__":
    cfg = _cfg("cfg3", name="cfg3_16k", n=16384)
    t0 = time.perf_counter()
    ck, _, t_comp = build(cfg, 1)
    a = marshal(ck)
    out = {k: a[k] for k in ("perm", "node_begin", "node_end", "node_left", "node_right", "rank", "skel_off", "skel")}
    out["coeff_norm"] = np.float64(np.linalg.norm(a["coeff"]))
    out["n"] = np.int64(cfg.n)
    np.savez_compressed(os.path.join(HERE, "producer16k.npz"), **out)
    print(f"cfg3 N=16384: {len(ck.tree.nodes)} nodes, ranks {sorted(set(a['rank'].tolist()))[:5]}, "
          f"compress {t_comp:.1f}s, total {time.perf_counter() - t0:.1f}s")
