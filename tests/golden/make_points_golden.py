"""Points file fixture written by the REFERENCE's save_points (points.py:76-88),
for the byte-compatibility test of paper_1602_01376_b200.persist.
Run in the build container: python tests/golden/make_points_golden.py"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
import kernelsolve as ks  # noqa: E402  (reference, build container only)

pts = ks.gen_synthetic("gaussian-mixture", 37, 5, seed=3)
ks.save_points(pts, os.path.join(HERE, "points_ref.f64"), "f64-binary")
np.save(os.path.join(HERE, "points_ref_coords.npy"), pts.coords)
print("points_ref.f64", os.path.getsize(os.path.join(HERE, "points_ref.f64")), "bytes")
