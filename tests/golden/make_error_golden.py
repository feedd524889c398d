"""Error-path fixtures made by running the REFERENCE `kernelsolve` package.

Run in the build container (needs /root/reference):
    python tests/golden/make_error_golden.py

Tiny operators that fail the way the reference reports it (the first two in a
reduced system Z, solver.py:138-149, with the failing node NOT the root; the third
in a leaf):

* singular.npz  -- two coincident points (exactly representable coordinates)
  are the skeletons of two sibling leaves, lambda = 0: the leaf blocks are
  exactly I, H = P P^T = [1], the coupling of the coincident skeleton points is
  exp(0) = 1, so the Z of their parent (node 1) is [[1, 1], [1, 1]] and the LU
  meets an exactly zero pivot column: SingularMatrixError (linalg.py:205-206).
* illcond_hard.npz -- the P of two sibling leaves is scaled so that
  det Z = 1 - B^2 H_l H_r = 1e-15 at their parent (node 2): the Hager estimate
  (linalg.py:282-304) is ~4e15 > 1e14 and the reference raises
  IllConditionedError(2, cond) (solver.py:150-152).

* leaf_not_spd.npz -- a leaf with two coincident points at lambda = 0: the Cholesky
  fails (NotSPDError), the LU fallback (solver.py:125-131) meets an exactly zero pivot
  column: SingularMatrixError raised from the leaf.

The tree and leaf blocks are the reference's own (build_tree, compress); the
rank-1 skeletons and P are set by hand and the couplings recomputed with the
reference's kernel_block, so the reference and the GPU consume the same arrays. Stored like make_golden.py's
fixtures plus expect_error, error_node and (ill-conditioned) error_cond.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import kernelsolve as ks  # noqa: E402  (reference, build container only)

from make_golden import int_hash, marshal  # noqa: E402


def _ck(x: np.ndarray, h: float):
    """Points on a line (second coordinate 0), leaf size 2: leaves hold
    consecutive pairs of the sorted x (tree.py:84-130). Far-apart pairs make
    every leaf block exactly the identity (exp(-|dx|^2/2h^2) underflows to 0)."""
    coords = np.stack([x, np.zeros_like(x)], axis=1)
    pts = ks.PointSet(coords)
    tree = ks.build_tree(pts, 2)
    spec = ks.KernelSpec("gaussian", bandwidth=h)
    params = ks.CompressParams(tol=1e-5, max_rank=1, n_neighbors=1, seed=0)
    return ks.compress(pts, tree, spec, params)


def _set_skeletons(ck, pick: dict[int, int], scale: dict[int, float]) -> None:
    """Rank-1 skeletons chosen by hand: leaf v keeps point pick[v] with
    coefficient scale[v] (default 1) on it and 0 on its other point; every
    internal node keeps its left child's skeleton point with coefficients
    [1, 0]. The couplings are recomputed from these skeletons with the
    reference's own kernel_block (compress.py:276-283)."""
    tree = ck.tree
    for nd in sorted(tree.nodes, key=lambda t: -t.level):
        if nd.size == ck.n:
            continue
        sk = ck.skeletons[nd.id]
        if nd.is_leaf:
            cand = tree.node_points(nd.id)
            j = int(np.nonzero(cand == pick[nd.id])[0][0])
            coeff = np.zeros((1, cand.size))
            coeff[0, j] = scale.get(nd.id, 1.0)
            sk.cand, sk.skel, sk.coeff = cand, np.array([pick[nd.id]], np.int64), coeff
        else:
            l, r = nd.children
            sk.cand = np.concatenate([ck.skeletons[l].skel, ck.skeletons[r].skel])
            sk.skel, sk.coeff = ck.skeletons[l].skel.copy(), np.array([[1.0, 0.0]])
    for nd in tree.nodes:
        if not nd.is_leaf:
            l, r = nd.children
            ck.couplings[nd.id] = ks.kernel_block(ck.spec, ck.points, ck.skeletons[l].skel, ck.skeletons[r].skel)


def _leaves(ck):
    return [nd for nd in ck.tree.nodes if nd.is_leaf]


def _save(name: str, ck, lam: float, exc) -> None:
    arrs = marshal(ck)
    arrs["lam"] = np.float64(lam)
    arrs["b"] = np.ones((ck.n, 1))
    arrs["int_hash"] = np.array(int_hash(arrs))
    arrs["expect_error"] = np.array(type(exc).__name__)
    arrs["error_node"] = np.int64(getattr(exc, "node_id", -1))
    arrs["error_cond"] = np.float64(getattr(exc, "cond_estimate", np.nan))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrs)
    print(f"{name}: reference raised {type(exc).__name__}: {exc}")


def make_singular() -> None:
    # sorted x: leaves {-100, 0} {0, 100} {200, 300} {400, 500}; points 1 and 2
    # coincide and are the skeletons of the sibling leaves 3 and 4
    x = np.array([-100.0, 0.0, 0.0, 100.0, 200.0, 300.0, 400.0, 500.0])
    ck = _ck(x, 1.0)
    lv = _leaves(ck)
    assert [nd.id for nd in lv] == [3, 4, 5, 6]
    pick = {3: 1, 4: 2, 5: 4, 6: 6}
    assert set(ck.tree.node_points(3)) == {0, 1} and set(ck.tree.node_points(4)) == {2, 3}
    _set_skeletons(ck, pick, {})
    try:
        ks.factorize(ck, 0.0)
    except ks.SingularMatrixError as exc:
        _save("singular", ck, 0.0, exc)
        return
    raise AssertionError("reference did not raise SingularMatrixError")


def make_illcond_hard() -> None:
    # sorted x: leaves {-300, -200} {-100, 0} {200, 300} {300.5, 400}; the
    # skeletons of leaves 5 and 6 are 300 and 300.5 (coupling b = exp(-1/8))
    x = np.array([-300.0, -200.0, -100.0, 0.0, 200.0, 300.0, 300.5, 400.0])
    h, lam, eps = 1.0, 0.0, 1e-15
    ck = _ck(x, h)
    assert [nd.id for nd in _leaves(ck)] == [3, 4, 5, 6]
    assert set(ck.tree.node_points(5)) == {4, 5} and set(ck.tree.node_points(6)) == {6, 7}
    b = float(np.exp(-0.25 / (2 * h * h)))
    p = ((1.0 - eps) / (b * b)) ** 0.25  # H = p^2 per leaf (A = I), det Z = 1 - b^2 p^4 = eps
    _set_skeletons(ck, {3: 0, 4: 3, 5: 5, 6: 6}, {5: p, 6: p})
    try:
        ks.factorize(ck, lam)
    except ks.IllConditionedError as exc:
        assert exc.node_id == 2
        _save("illcond_hard", ck, lam, exc)
        return
    raise AssertionError("reference did not raise IllConditionedError")


def make_leaf_not_spd() -> None:
    # sorted x: leaves {0, 0} {100, 101} {200, 201} {300, 301}: the first leaf holds
    # two coincident points, so at lambda = 0 its block is exactly [[1, 1], [1, 1]]:
    # _cholesky meets the pivot 1 - 1*1 = 0 (NotSPDError, linalg.py:190-192), factorize
    # falls back to the pivoted LU (solver.py:125-131), whose second column is exactly
    # zero: SingularMatrixError (linalg.py:205-206) from the LEAF. No rounding is
    # involved, so the GPU must detect the same pivot in its blocked Cholesky.
    x = np.array([0.0, 0.0, 100.0, 101.0, 200.0, 201.0, 300.0, 301.0])
    ck = _ck(x, 1.0)
    lv = _leaves(ck)
    assert [nd.id for nd in lv] == [3, 4, 5, 6]
    assert set(ck.tree.node_points(3)) == {0, 1}
    _set_skeletons(ck, {3: 0, 4: 2, 5: 4, 6: 6}, {})
    try:
        ks.factorize(ck, 0.0)
    except ks.SingularMatrixError as exc:
        assert "elimination step 1" in str(exc)
        _save("leaf_not_spd", ck, 0.0, exc)
        return
    raise AssertionError("reference did not raise SingularMatrixError")


if __name__ == "__main__":
    make_singular()
    make_illcond_hard()
    make_leaf_not_spd()
