"""Independent checks written straight from the definitions, for pinning the oracle.

* ``chordless_cycles_brute``: the plain definition (§1): S subset of V with
  |S| >= 3 is a chordless cycle iff G[S] is connected and 2-regular.  Exhaustive over all
  2^n subsets -- no labelling, no triplets, no DFS.
* ``hspec_hash``: the set hash of DESIGN.md "H-spec" recomputed in Python from a list of
  vertex sets (cross-implementation check of the C oracle's hashing).
"""
import itertools

M64 = (1 << 64) - 1
DEFAULT_SEED = 0x1410487600000000


def adjacency_sets(n, row_ptr, col):
    return [set(int(c) for c in col[row_ptr[v]:row_ptr[v + 1]]) for v in range(n)]


def _is_chordless_cycle(S, adj):
    S = set(S)
    for v in S:
        if len(adj[v] & S) != 2:
            return False
    # connected?
    start = next(iter(S))
    seen = {start}
    stack = [start]
    while stack:
        v = stack.pop()
        for w in adj[v] & S:
            if w not in seen:
                seen.add(w)
                stack.append(w)
    return len(seen) == len(S)


def chordless_cycles_brute(n, row_ptr, col):
    """All vertex sets of chordless cycles, as frozensets.  Feasible for n <= ~18."""
    adj = adjacency_sets(n, row_ptr, col)
    out = set()
    for mask in range(1 << n):
        if bin(mask).count("1") < 3:
            continue
        S = [v for v in range(n) if (mask >> v) & 1]
        # quick degree filter
        ok = True
        Ss = set(S)
        for v in S:
            if len(adj[v] & Ss) != 2:
                ok = False
                break
        if ok and _is_chordless_cycle(S, adj):
            out.add(frozenset(S))
    return out


def splitmix_finaliser(x):
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def hspec_hash(vertex_sets, seed=DEFAULT_SEED):
    total = 0
    for S in vertex_sets:
        s = 0
        for v in S:
            s = (s + splitmix_finaliser(seed ^ v)) & M64
        total = (total + splitmix_finaliser(s)) & M64
    return total


def counts_of(vertex_sets, n):
    c = [0] * (n + 1)
    for S in vertex_sets:
        c[len(S)] += 1
    return c


def comb(a, b):
    if b < 0 or a < b:
        return 0
    from math import comb as _c
    return _c(a, b)


def hspec_hash_np(vertices, offsets, seed=DEFAULT_SEED):
    """hspec_hash over many cycles at once (numpy, uint64 arithmetic wraps mod 2^64):
    vertices int32[], offsets uint64[k+1] as returned by cc_fetch_cycles."""
    import numpy as np

    def mix(x):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))

    with np.errstate(over="ignore"):
        keys = mix(np.uint64(seed) ^ vertices.astype(np.uint64))
        starts = offsets[:-1].astype(np.int64)
        sums = np.add.reduceat(keys, starts) if len(starts) else np.zeros(0, np.uint64)
        return int(mix(sums).sum(dtype=np.uint64))
