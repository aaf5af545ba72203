"""O1 — basic and composite partitions (Def. partitions PAPER.md:230-242,
Fig. basic/composite PAPER.md:247-252, App. A.2).

Test infrastructure (see oracle/__init__.py).

Basic cells: s x s pixel blocks, i = i1 * n2 + i2.
A-partition: 2x2 groups {2j1, 2j1+1} x {2j2, 2j2+1} (clipped at the far border
if n is odd).
B-partition: groups offset by one basic cell, {2j1-1, 2j1} x {2j2-1, 2j2},
intersected with the grid; border groups are ragged (2x1, 1x2, 1x1) instead
of the paper's padding (reading R4).
Members are listed in row-major basic-cell order.
"""
from __future__ import annotations

from collections import deque

import numpy as np


def basic_partition(mu: np.ndarray, s: int):
    """Basic cell masses m_i = mu(X_i) (Def. partitions)."""
    N1, N2 = mu.shape
    assert N1 % s == 0 and N2 % s == 0
    n1, n2 = N1 // s, N2 // s
    m = mu.reshape(n1, s, n2, s).sum(axis=(1, 3)).ravel()
    if np.any(m <= 0):
        raise ValueError("zero-mass basic cell (PAPER.md:233 requires m_i > 0)")
    return n1, n2, m


def composite_partition(n1: int, n2: int, kind: str):
    """List of composite cells; each is a list of basic-cell indices in
    row-major order."""
    if kind == "A":
        rows = [[r for r in (2 * j, 2 * j + 1) if r < n1] for j in range((n1 + 1) // 2)]
        cols = [[c for c in (2 * j, 2 * j + 1) if c < n2] for j in range((n2 + 1) // 2)]
    elif kind == "B":
        rows = [[r for r in (2 * j - 1, 2 * j) if 0 <= r < n1] for j in range(n1 // 2 + 1)]
        cols = [[c for c in (2 * j - 1, 2 * j) if 0 <= c < n2] for j in range(n2 // 2 + 1)]
        rows = [r for r in rows if r]
        cols = [c for c in cols if c]
    else:
        raise ValueError(kind)
    cells = []
    for rr in rows:
        for cc in cols:
            cells.append([r * n2 + c for r in rr for c in cc])
    return cells


def partition_graph_connected(n1: int, n2: int, A=None, B=None) -> bool:
    """Def. PartitionGraph: vertices = A and B composite
    cells, edge iff they share a basic cell.  BFS connectivity.  A and B
    default to the staggered grid partitions; explicit partitions (lists of
    basic-cell index lists) may be given."""
    A = composite_partition(n1, n2, "A") if A is None else A
    B = composite_partition(n1, n2, "B") if B is None else B
    verts = [("A", k) for k in range(len(A))] + [("B", k) for k in range(len(B))]
    owner = {}
    for k, J in enumerate(A):
        for i in J:
            owner.setdefault(i, []).append(("A", k))
    for k, J in enumerate(B):
        for i in J:
            owner.setdefault(i, []).append(("B", k))
    adj = {v: set() for v in verts}
    for lst in owner.values():
        for u in lst:
            for v in lst:
                if u != v:
                    adj[u].add(v)
    seen = {verts[0]}
    dq = deque([verts[0]])
    while dq:
        u = dq.popleft()
        for v in adj[u]:
            if v not in seen:
                seen.add(v)
                dq.append(v)
    return len(seen) == len(verts)


def cell_pixels(i: int, n2: int, s: int):
    """Pixel (row, col) arrays of basic cell X_i, row-major."""
    i1, i2 = divmod(i, n2)
    r, c = np.meshgrid(np.arange(i1 * s, (i1 + 1) * s), np.arange(i2 * s, (i2 + 1) * s), indexing="ij")
    return r.ravel(), c.ravel()
