"""Restatement of the reference partition tree (tree.py:84-130) for operator
production at sizes where running the reference is impractical.

Same rule, same bits: split the coordinate of maximum spread (lowest axis on
ties) at the stable-sort median, mid = (size + 1) // 2, breadth-first ids.
`tests/test_producer.py` checks perm and node table against the reference's
own trees stored in the golden fixtures.
"""

from __future__ import annotations

import numpy as np


def build_tree(coords: np.ndarray, leaf_size: int) -> dict:
    if leaf_size < 2:
        raise ValueError(f"leaf_size must be >= 2, got {leaf_size}")
    n = coords.shape[0]
    perm = np.arange(n, dtype=np.int64)
    begin, end, level, left, right = [], [], [], [], []
    queue = [(0, n, 0, -1)]
    head = 0
    while head < len(queue):
        b, e, lev, parent = queue[head]
        head += 1
        nid = len(begin)
        begin.append(b)
        end.append(e)
        level.append(lev)
        left.append(-1)
        right.append(-1)
        if parent >= 0:
            if left[parent] < 0:
                left[parent] = nid
            else:
                right[parent] = nid
        size = e - b
        if size <= leaf_size:
            continue
        local = coords[perm[b:e]]
        spans = local.max(axis=0) - local.min(axis=0)
        axis = int(np.argmax(spans))
        order = np.argsort(local[:, axis], kind="stable")
        perm[b:e] = perm[b:e][order]
        mid = (size + 1) // 2
        queue.append((b, b + mid, lev + 1, nid))
        queue.append((b + mid, e, lev + 1, nid))
    return {
        "perm": perm,
        "node_begin": np.array(begin, np.int64),
        "node_end": np.array(end, np.int64),
        "node_level": np.array(level, np.int64),
        "node_left": np.array(left, np.int64),
        "node_right": np.array(right, np.int64),
    }
