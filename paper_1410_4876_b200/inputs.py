"""Seeded synthetic input graphs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no labelling, no triplets, no chord test,
no hashing).  It only builds undirected simple graphs in CSR form:
``(n, row_ptr: int64[n+1], col: int32[2m])`` with every neighbour block sorted ascending.

Families follow the paper's synthetic Table 1 rows (§5) and the
BASELINE.json configs; vertex numbering follows SPEC.md:74,109 (row-major grids, hub last):

* ``grid(r, c)``            P_r x P_c, id = c*row + col
* ``complete_bipartite(a,b)`` A = 0..a-1, B = a..a+b-1
* ``cycle(k)``              C_k on 0..k-1
* ``wheel(k)``              rim 0..k-1, hub k
* ``complete(k)``, ``path(k)``, ``star(k)``, ``random_tree(n, seed)``      closed-form pins
* ``gnp(n, p, seed)``        Erdos-Renyi G(n, p) from numpy's PCG64 stream  (BASELINE configs[3])
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "edges_to_csr", "csr_to_edges", "grid", "complete_bipartite", "cycle", "wheel",
    "complete", "path", "star", "random_tree", "gnp", "permute", "fig1_graph", "named",
]


def edges_to_csr(n: int, edges) -> tuple[int, np.ndarray, np.ndarray]:
    """Symmetrise an undirected edge list into sorted CSR (duplicates merged)."""
    e = np.asarray(list(edges) if not isinstance(edges, np.ndarray) else edges, dtype=np.int64)
    if e.size == 0:
        return n, np.zeros(n + 1, dtype=np.int64), np.zeros(0, dtype=np.int32)
    e = e.reshape(-1, 2)
    if (e < 0).any() or (e >= n).any():
        raise ValueError("edge endpoint out of range")
    if (e[:, 0] == e[:, 1]).any():
        raise ValueError("self-loop")
    both = np.concatenate([e, e[:, ::-1]], axis=0)
    key = np.unique(both[:, 0] * n + both[:, 1])
    src = key // n
    dst = key % n
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(row_ptr, src + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    return n, row_ptr.astype(np.int64), dst.astype(np.int32)


def csr_to_edges(n, row_ptr, col) -> np.ndarray:
    src = np.repeat(np.arange(n, dtype=np.int64), np.diff(row_ptr))
    dst = np.asarray(col, dtype=np.int64)
    m = src < dst
    return np.stack([src[m], dst[m]], axis=1)


def grid(r: int, c: int):
    """P_r x P_c grid graph, vertex (i, j) -> id c*i + j (row-major)."""
    edges = []
    for i in range(r):
        for j in range(c):
            v = c * i + j
            if j + 1 < c:
                edges.append((v, v + 1))
            if i + 1 < r:
                edges.append((v, v + c))
    return edges_to_csr(r * c, edges)


def complete_bipartite(a: int, b: int):
    edges = [(i, a + j) for i in range(a) for j in range(b)]
    return edges_to_csr(a + b, edges)


def cycle(k: int):
    return edges_to_csr(k, [(i, (i + 1) % k) for i in range(k)])


def wheel(k: int):
    """W_k: rim cycle 0..k-1 plus hub k joined to every rim vertex."""
    edges = [(i, (i + 1) % k) for i in range(k)] + [(i, k) for i in range(k)]
    return edges_to_csr(k + 1, edges)


def complete(k: int):
    return edges_to_csr(k, [(i, j) for i in range(k) for j in range(i + 1, k)])


def path(k: int):
    return edges_to_csr(k, [(i, i + 1) for i in range(k - 1)])


def star(k: int):
    """K_{1,k} with hub 0."""
    return edges_to_csr(k + 1, [(0, i) for i in range(1, k + 1)])


def random_tree(n: int, seed: int):
    rng = np.random.default_rng(seed)
    edges = [(int(rng.integers(0, i)), i) for i in range(1, n)]
    return edges_to_csr(n, edges)


def gnp(n: int, p: float, seed: int):
    """Erdos-Renyi G(n, p): each pair i<j is an edge iff a PCG64 uniform draw < p.

    The draws are taken row by row (i ascending, j>i ascending) from
    ``numpy.random.default_rng(seed)`` so the graph is a pure function of (n, p, seed).
    """
    rng = np.random.default_rng(seed)
    edges = []
    for i in range(n - 1):
        u = rng.random(n - 1 - i)
        js = np.nonzero(u < p)[0] + i + 1
        if js.size:
            edges.append(np.stack([np.full(js.size, i, dtype=np.int64), js.astype(np.int64)], axis=1))
    if not edges:
        return edges_to_csr(n, [])
    return edges_to_csr(n, np.concatenate(edges, axis=0))


def permute(n, row_ptr, col, perm):
    """Relabel vertex v as perm[v]; returns a new CSR of the isomorphic graph."""
    perm = np.asarray(perm, dtype=np.int64)
    e = csr_to_edges(n, row_ptr, col)
    return edges_to_csr(n, perm[e])


def fig1_graph():
    """A graph consistent with the caption of Fig. 1: vertex 0 is adjacent to
    1 and 3, vertex 1 to 0, 2 and 4 (the remaining edges of the figure are not in the text;
    two are added so the graph has a cycle: 2-5, 4-5, 3-4)."""
    return edges_to_csr(6, [(0, 1), (0, 3), (1, 2), (1, 4), (2, 5), (4, 5), (3, 4)])


# Named BASELINE.json workloads (configs[0..4]) and the Table-1 synthetic rows.
def named(name: str):
    name = name.lower()
    if name in ("p4x4", "grid4x4"):
        return grid(4, 4)
    if name in ("k150", "k150x150", "k_150_150"):
        return complete_bipartite(150, 150)
    if name in ("p8x8", "grid8x8"):
        return grid(8, 8)
    if name in ("p10x10", "grid10x10"):
        return grid(10, 10)
    if name in ("gnp2000", "g2000"):
        return gnp(2000, 0.005, GNP_SEED)
    if name.startswith("grid") and "x" in name:
        a, b = name[4:].split("x")
        return grid(int(a), int(b))
    if name.startswith("k") and "x" in name:
        a, b = name[1:].split("x")
        return complete_bipartite(int(a), int(b))
    if name.startswith("c") and name[1:].isdigit():
        return cycle(int(name[1:]))
    if name.startswith("wheel"):
        return wheel(int(name[5:]))
    raise KeyError(name)


GNP_SEED = 14104876
