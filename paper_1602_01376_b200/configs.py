"""The five BASELINE.json configurations and their seeded point recipes.

Recipes follow SURVEY.md §8(d). Config 1 is the reference's own
`gen_synthetic("uniform-cube", 4096, 8, seed=0)` (`points.py:132-163`);
configs 2-5 have no generator in the reference, so their recipes are the
survey's, drawn from the reference RNG (`rng.py:36-38`) with root seed 0.
The RHS is `generator(0, 0x726873).standard_normal(...)` (the `cli.py:38,270`
tag), permuted into tree order by the caller.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from .rng import generator

_UNIFORM_CUBE_TAG = 0x6375  # points.py:20
RHS_TAG = 0x726873  # cli.py:38


@dataclass(frozen=True)
class Config:
    name: str
    recipe: str
    n: int
    d: int
    h: float
    lam: float
    leaf_size: int
    max_rank: int
    q: tuple[int, ...]
    tol_u: float  # relative L2 tolerance on u (north_star)
    tol: float = 1e-5  # CompressParams defaults (compress.py:49-53)
    n_neighbors: int = 32
    seed: int = 0

    def scaled(self, n: int, leaf_size: int | None = None, max_rank: int | None = None,
               suffix: str = "s") -> "Config":
        """Same recipe/kernel/lambda at a reduced size (for fixtures and tests)."""
        return replace(self, name=self.name + suffix, n=n,
                       leaf_size=leaf_size or self.leaf_size,
                       max_rank=max_rank or self.max_rank)


CONFIGS = {
    "cfg1": Config("cfg1", "cfg1", 4096, 8, 0.5, 1.0, 128, 64, (1,), 1e-10),
    "cfg2": Config("cfg2", "cfg2", 65536, 18, 1.0, 0.1, 512, 128, (1,), 1e-10),
    "cfg3": Config("cfg3", "cfg3", 1048576, 28, 1.5, 0.1, 1024, 256, (1, 32), 1e-10),
    "cfg4": Config("cfg4", "cfg4", 524288, 54, 0.8, 1.0, 512, 256, (16,), 1e-10),
    "cfg5": Config("cfg5", "cfg5", 2097152, 784, 0.3, 0.01, 2048, 512, (1,), 1e-8),
}


def gen_points(cfg: Config) -> np.ndarray:
    """Points in ORIGINAL order, (n, d) float64, per SURVEY.md §8(d)."""
    base = cfg.recipe
    n, d = cfg.n, cfg.d
    if base == "cfg1":
        # points.py:151-152 (gen_synthetic uniform-cube)
        return generator(cfg.seed, _UNIFORM_CUBE_TAG).uniform(0.0, 1.0, size=(n, d))
    if base == "cfg2":
        rng = generator(cfg.seed, 0xB5E2)
        means = rng.uniform(-3.0, 3.0, (8, d))
        assign = rng.integers(0, 8, n)
        return means[assign] + rng.standard_normal((n, d))
    if base == "cfg3":
        rng = generator(cfg.seed, 0xB5E3)
        scales = rng.uniform(0.5, 2.0, d)
        return rng.standard_normal((n, d)) * scales
    if base == "cfg4":
        rng = generator(cfg.seed, 0xB5E4)
        c = rng.standard_normal((n, 10))
        b = (rng.random((n, d - 10)) < 0.1).astype(np.float64)
        return np.hstack([c, b])
    if base == "cfg5":
        rng = generator(cfg.seed, 0xB5E5)
        x = rng.uniform(0.0, 1.0, (n, d))
        x[rng.random((n, d)) < 0.7] = 0.0
        nrm = np.sqrt(np.einsum("ij,ij->i", x, x))
        nrm[nrm == 0.0] = 1.0
        return x / nrm[:, None]
    raise ValueError(f"unknown config {cfg.name}")


def gen_rhs(cfg: Config, q: int) -> np.ndarray:
    """RHS in ORIGINAL order: (n,) for q == 0 sentinel-free 1-RHS use, else (n, q)."""
    rng = generator(cfg.seed, RHS_TAG)
    if q == 1:
        return rng.standard_normal(cfg.n)
    return rng.standard_normal((cfg.n, q))
