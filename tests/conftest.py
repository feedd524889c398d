import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libinvaskit.so")
    config.addinivalue_line("markers", "slow: larger CPU oracle cases")


def load_golden(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False) as z:
        g = {k: z[k] for k in z.files}
    if "coords" not in g and "gen_cfg" in g:
        # large fixtures do not carry their points: regenerate them from the
        # recipe (configs.gen_points) and check the bits against the reference's
        import hashlib
        import json

        from paper_1602_01376_b200.configs import Config, gen_points

        kw = json.loads(str(g["gen_cfg"]))
        kw["q"] = tuple(kw["q"])
        c = np.ascontiguousarray(gen_points(Config(**kw)), dtype="<f8")
        assert hashlib.sha256(c.tobytes()).hexdigest() == str(g["coords_sha256"]), "point recipe drifted"
        g["coords"] = c
    return g


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = load_golden(name)
        return cache[name]

    return get


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
