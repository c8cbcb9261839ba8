"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Integer method: every comparison is bit-exact -- per-length counts, the 64-bit set
hash, |F_t| per level, candidate slots, and (collect mode) the canonical cycle sequences.
"""
import math
import os

import numpy as np
import pytest

import oracle
from paper_1410_4876_b200 import binding, build, inputs as I
from tests import brute

pytestmark = pytest.mark.gpu

NT = os.cpu_count() or 1


@pytest.fixture(scope="module")
def ws():
    import torch
    assert torch.cuda.is_available()
    build.build()
    binding.load()
    return torch.empty(1 << 30, dtype=torch.uint8, device="cuda")


def gpu(g, ws, **kw):
    return binding.enumerate_cycles(*g, workspace=ws, **kw)


def assert_same(got, want, paths=True):
    assert got["counts"].tolist() == want["counts"].tolist()
    assert got["set_hash"] == want["set_hash"]
    if paths:
        assert got["paths_by_len"].tolist() == want["paths_by_len"].tolist()
        assert got["candidates"] == want["candidates"]


SMALL = [
    ("p4x4", I.grid(4, 4)), ("p3x5", I.grid(3, 5)), ("k3x4", I.complete_bipartite(3, 4)),
    ("k5", I.complete(5)), ("k12", I.complete(12)), ("c3", I.cycle(3)), ("c7", I.cycle(7)),
    ("w6", I.wheel(6)), ("w3", I.wheel(3)), ("fig1", I.fig1_graph()), ("path5", I.path(5)),
    ("star4", I.star(4)), ("tree40", I.random_tree(40, 3)), ("empty5", I.edges_to_csr(5, [])),
    ("empty0", I.edges_to_csr(0, [])), ("one", I.edges_to_csr(1, [])), ("edge", I.edges_to_csr(2, [(0, 1)])),
    ("two_triangles", I.edges_to_csr(7, [(0, 1), (1, 2), (2, 0), (4, 5), (5, 6), (6, 4)])),
] + [(f"gnp{n}_{p}_{s}", I.gnp(n, p, 7000 + 31 * n + s)) for n in (8, 12, 16, 24) for p in (0.2, 0.35, 0.5)
     for s in range(2)]


@pytest.mark.parametrize("name,g", SMALL, ids=[s[0] for s in SMALL])
def test_small_graphs_collect(ws, name, g):
    got = gpu(g, ws, collect=True)
    want = oracle.enumerate_cycles(*g, collect=True)
    assert_same(got, want)
    # same labelling (lowest-id ties) on both sides -> identical canonical sequences
    assert sorted(map(tuple, got["cycles"])) == sorted(map(tuple, want["cycles"]))


def test_p4x4_config0_full_list_vs_brute_force(ws):
    """BASELINE configs[0]: P4xP4 full chordless-cycle list vs oracle and brute force."""
    g = I.grid(4, 4)
    got = gpu(g, ws, collect=True)
    assert {k: int(v) for k, v in enumerate(got["counts"]) if v} == {4: 9, 8: 4, 10: 4, 12: 7}
    assert {frozenset(c) for c in got["cycles"]} == brute.chordless_cycles_brute(*g)
    assert got["set_hash"] == brute.hspec_hash(brute.chordless_cycles_brute(*g))


TABLE1 = [("C_100", I.cycle(100), 1), ("Wheel_100", I.wheel(100), 101),
          ("K_8_8", I.complete_bipartite(8, 8), 784), ("K_50_50", I.complete_bipartite(50, 50), 1500625),
          ("Grid_4x10", I.grid(4, 10), 1823), ("Grid_5x6", I.grid(5, 6), 749),
          ("Grid_5x10", I.grid(5, 10), 52620), ("Grid_6x6", I.grid(6, 6), 3436),
          ("Grid_6x10", I.grid(6, 10), 800139), ("Grid_7x10", I.grid(7, 10), 8136453)]


@pytest.mark.parametrize("name,g,total", TABLE1, ids=[t[0] for t in TABLE1])
def test_table1_graphs(ws, name, g, total):
    """Table 1 synthetic rows: totals from the paper, everything else
    (per-length counts, hash, |F_t|, candidates) from the oracle."""
    got = gpu(g, ws)
    assert int(got["counts"].sum()) == total
    assert_same(got, oracle.enumerate_cycles(*g, nthreads=NT))


def test_k150_config1(ws):
    """BASELINE configs[1]: K_{150,150} -> C(150,2)^2 = 124,880,625 4-cycles; |F_3| = 1,113,775
    and 167,066,250 candidate slots; hash vs oracle."""
    g = I.complete_bipartite(150, 150)
    got = gpu(g, ws)
    assert int(got["counts"][4]) == math.comb(150, 2) ** 2 == int(got["counts"].sum())
    assert int(got["paths_by_len"][3]) == 1113775
    assert got["candidates"] == 167066250
    assert_same(got, oracle.enumerate_cycles(*g, nthreads=NT))


def test_p8x8_config2(ws):
    """BASELINE configs[2]: P8x8, full enumeration; N4..N12 closed forms + oracle."""
    g = I.grid(8, 8)
    got = gpu(g, ws)
    c = got["counts"]
    assert [int(c[k]) for k in (4, 6, 8, 10, 12)] == [49, 0, 36, 60, 223]
    assert_same(got, oracle.enumerate_cycles(*g, nthreads=NT))


@pytest.mark.parametrize("K", [14, 18, 22])
def test_p10x10_config4_capped(ws, K):
    """BASELINE configs[4] at full graph size with a length cap (the oracle finishes in < 1 s):
    per-length counts, hash and |F_t| for k <= K; N4..N12 closed forms."""
    g = I.grid(10, 10)
    got = gpu(g, ws, max_len=K)
    c = got["counts"]
    assert [int(c[k]) for k in (4, 6, 8, 10, 12)] == [81, 0, 64, 112, 439]
    assert_same(got, oracle.enumerate_cycles(*g, max_len=K, nthreads=NT))


@pytest.mark.parametrize("K", [3, 4, 5, 6, 7])
def test_gnp_dense_capped(ws, K):
    """G(n, p) with n in the bitmap class (n = 500 -> 8 words) and a length cap."""
    g = I.gnp(500, 0.02, 11)
    assert_same(gpu(g, ws, max_len=K), oracle.enumerate_cycles(*g, max_len=K, nthreads=NT))


@pytest.mark.parametrize("n", [63, 64, 65, 127, 128, 129, 191, 200, 256, 300, 383, 448, 511, 512])
def test_word_boundaries(ws, n):
    """Every bitmap width NW = 1..8 and the word boundaries (vertex 63/64 etc.)."""
    g = I.gnp(n, 3.0 / n, 100 + n)
    assert_same(gpu(g, ws, max_len=12), oracle.enumerate_cycles(*g, max_len=12, nthreads=NT))


def test_dense_random_warp_variant(ws):
    """Delta > 32 selects the warp-per-path kernel; check it on a graph with long paths too."""
    g = I.gnp(120, 0.35, 5)
    assert int(np.diff(g[1]).max()) > 32
    assert_same(gpu(g, ws, max_len=6), oracle.enumerate_cycles(*g, max_len=6, nthreads=NT))
    g = I.wheel(60)
    assert_same(gpu(g, ws), oracle.enumerate_cycles(*g))


@pytest.mark.parametrize("K", [3, 4, 5, 8, 10, 13])
def test_max_len(ws, K):
    g = I.grid(5, 6)
    assert_same(gpu(g, ws, max_len=K), oracle.enumerate_cycles(*g, max_len=K))


@pytest.mark.parametrize("pages", [64, 96, 128, 4096])
def test_chunked_scheduler_matches_level_synchronous(ws, pages):
    """A small workspace forces the depth-first chunk scheduler (PAPER.md:455 future work);
    results must be identical to the oracle.  P7xP8: n = 56 (12-byte records, 1024-record
    pages of 12 KiB), peak frontier 444,975 paths -- 64..128 pages cannot hold it."""
    import torch
    g = I.grid(7, 8)
    small = torch.empty(pages * 1024 * 12, dtype=torch.uint8, device="cuda")
    got = binding.enumerate_cycles(*g, workspace=small)
    st = got["stats"]
    if pages <= 128:
        assert st["chunks"] > st["rounds"]
        assert st["peak_arena_records"] <= st["arena_capacity"] < 444975
    want = oracle.enumerate_cycles(*g, nthreads=NT)
    assert_same(got, want)
    if pages in (64, 4096):
        got_c = binding.enumerate_cycles(*g, workspace=small, collect=True)
        want_c = oracle.enumerate_cycles(*g, collect=True)
        assert sorted(map(tuple, got_c["cycles"])) == sorted(map(tuple, want_c["cycles"]))


def test_chunked_k50(ws):
    import torch
    g = I.complete_bipartite(50, 50)
    small = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    got = binding.enumerate_cycles(*g, workspace=small)
    assert got["stats"]["chunks"] > 2
    assert_same(got, oracle.enumerate_cycles(*g, nthreads=NT))


def test_chunked_gnp_small_workspace(ws):
    """G(100, 0.1) capped at 9 vertices: |F_7| = 156,775 records do not fit a 1 MB arena, so the
    deepest-first chunk scheduler must split levels; the result is unchanged."""
    import torch
    g = I.gnp(100, 0.1, 4242)
    small = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    got = binding.enumerate_cycles(*g, workspace=small, max_len=9)
    assert got["stats"]["chunks"] > 2
    assert_same(got, oracle.enumerate_cycles(*g, max_len=9, nthreads=NT))


def test_workspace_too_small_fails_loudly(ws):
    import torch
    small = torch.empty(64 * 12, dtype=torch.uint8, device="cuda")
    with pytest.raises(binding.CCError) as ei:
        binding.enumerate_cycles(*I.complete_bipartite(50, 50), workspace=small)
    assert ei.value.kind == "CC_ERR_CAPACITY"


@pytest.mark.parametrize("W", [2, 3, 8])
@pytest.mark.parametrize("name,g", [("grid6x7", I.grid(6, 7)), ("k40", I.complete_bipartite(40, 40)),
                                    ("gnp", I.gnp(200, 0.04, 3))])
def test_shards_sum_to_the_whole(ws, W, name, g):
    """Shard-sum invariance: running shard_index = 0..W-1 and summing gives the
    unsharded counts, hash, |F_t| and candidates exactly."""
    kw = dict(max_len=9) if name == "gnp" else {}
    full = gpu(g, ws, **kw)
    parts = [gpu(g, ws, shard_index=i, shard_count=W, min_shard_paths=16, **kw) for i in range(W)]
    assert sum(p["counts"] for p in parts).tolist() == full["counts"].tolist()
    assert sum(p["set_hash"] for p in parts) % (1 << 64) == full["set_hash"]
    assert sum(p["paths_by_len"] for p in parts).tolist() == full["paths_by_len"].tolist()
    assert sum(p["candidates"] for p in parts) == full["candidates"]
    # every shard got real work
    assert all(int(p["paths_by_len"].sum()) > 0 for p in parts)


@pytest.mark.parametrize("stride", [2, 5, 9])
def test_root_sampling_matches_oracle(ws, stride):
    """Root samples are defined on original ids on both sides."""
    g = I.grid(7, 7)
    for off in range(stride):
        got = gpu(g, ws, root_stride=stride, root_offset=off)
        want = oracle.enumerate_cycles(*g, root_stride=stride, root_offset=off, nthreads=NT)
        assert_same(got, want)


def test_hash_seed(ws):
    g = I.grid(5, 5)
    assert_same(gpu(g, ws, hash_seed=99), oracle.enumerate_cycles(*g, seed=99))


def test_unsorted_rows_and_permuted_ids(ws):
    """Input normalisation + isomorphism: a permuted graph gives the permuted cycle sets."""
    n, rp, col = I.grid(5, 5)
    perm = np.random.default_rng(3).permutation(n)
    g2 = I.permute(n, rp, col, perm)
    a = gpu((n, rp, col), ws, collect=True)
    b = gpu(g2, ws, collect=True)
    assert {frozenset(int(perm[v]) for v in c) for c in a["cycles"]} == {frozenset(c) for c in b["cycles"]}
    # shuffle each row
    rng = np.random.default_rng(4)
    col3 = col.copy()
    for v in range(n):
        rng.shuffle(col3[rp[v]:rp[v + 1]])
    assert_same(gpu((n, rp, col3), ws), oracle.enumerate_cycles(n, rp, col))


def test_too_large_graph_rejected(ws):
    g = I.gnp(2016, 0.002, 1)
    with pytest.raises(binding.CCError) as ei:
        gpu(g, ws)
    assert ei.value.kind == "CC_ERR_TOO_LARGE"
    # collect mode above n = 512 needs the list records (a length cap 4..14, max degree <= 32)
    with pytest.raises(binding.CCError) as ei:
        gpu(I.gnp(600, 0.005, 1), ws, collect=True)
    assert ei.value.kind == "CC_ERR_TOO_LARGE"
    with pytest.raises(binding.CCError) as ei:
        gpu(I.gnp(600, 0.005, 1), ws, collect=True, max_len=8, record_format=1)
    assert ei.value.kind == "CC_ERR_TOO_LARGE"


# ---------------------------------------------------------------- wide class (512 < n <= 2015)
@pytest.mark.parametrize("K", [3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("fmt", [1, 2])
def test_gnp2000_config3_capped(ws, K, fmt):
    """BASELINE configs[3]: G(2000, 0.005) (seed inputs.GNP_SEED) per-length counts + set hash
    with a length cap (full enumeration is infeasible: ~1e190 cycles), in both
    frontier record formats (1 = blocked set, 2 = vertex list)."""
    g = I.gnp(2000, 0.005, I.GNP_SEED)
    if fmt == 2 and K < 4:
        with pytest.raises(binding.CCError) as ei:
            gpu(g, ws, max_len=K, record_format=2)
        assert ei.value.kind == "CC_ERR_INVALID_ARGUMENT"
        return
    got = gpu(g, ws, max_len=K, record_format=fmt)
    if K >= 4:
        assert got["stats"]["record_bytes"] == (32 if fmt == 2 else 264)
    assert_same(got, oracle.enumerate_cycles(*g, max_len=K, nthreads=NT))


@pytest.mark.parametrize("n,p,K", [(513, 0.02, 7), (600, 0.01, 9), (1024, 0.006, 8), (1500, 0.004, 9),
                                   (2015, 0.003, 9)])
@pytest.mark.parametrize("fmt", [1, 0])
def test_wide_class_sizes(ws, n, p, K, fmt):
    g = I.gnp(n, p, 4000 + n)
    assert_same(gpu(g, ws, max_len=K, record_format=fmt), oracle.enumerate_cycles(*g, max_len=K, nthreads=NT))


@pytest.mark.parametrize("K", [4, 5, 6, 11, 12, 13, 14])
def test_list_class_lengths(ws, K):
    """Vertex-list records across the id-word boundaries (t = 4, 8, 12 vertices per path) and up
    to the largest max_len the format takes (14: paths of 12 vertices, three id words)."""
    g = I.grid(24, 24)  # n = 576 > 512: wide; Delta = 4; long chordless paths
    got = gpu(g, ws, max_len=K, record_format=2)
    assert got["stats"]["record_bytes"] == (32 if K <= 10 else 40)
    assert_same(got, oracle.enumerate_cycles(*g, max_len=K, nthreads=NT))


def test_list_class_rejects_what_it_cannot_hold(ws):
    with pytest.raises(binding.CCError):
        gpu(I.grid(24, 24), ws, max_len=15, record_format=2)  # 13-vertex paths
    with pytest.raises(binding.CCError):
        gpu(I.gnp(700, 0.06, 3), ws, max_len=6, record_format=2)  # Delta > 32
    with pytest.raises(binding.CCError):
        gpu(I.grid(10, 10), ws, max_len=6, record_format=2)  # n <= 512


def test_wide_class_dense_and_grid(ws):
    """Wide class on a denser random graph (closures every level) and on a long-path graph."""
    g = I.gnp(700, 0.05, 9)
    assert_same(gpu(g, ws, max_len=5), oracle.enumerate_cycles(*g, max_len=5, nthreads=NT))
    g = I.grid(24, 24)  # n = 576, long chordless paths
    assert_same(gpu(g, ws, max_len=16), oracle.enumerate_cycles(*g, max_len=16, nthreads=NT))


@pytest.mark.parametrize("W", [2, 5])
@pytest.mark.parametrize("fmt", [1, 2])
def test_wide_class_shards(ws, W, fmt):
    g = I.gnp(2000, 0.005, I.GNP_SEED)
    full = gpu(g, ws, max_len=7, record_format=fmt)
    parts = [gpu(g, ws, max_len=7, shard_index=i, shard_count=W, record_format=fmt, min_shard_paths=256)
             for i in range(W)]
    assert sum(p["counts"] for p in parts).tolist() == full["counts"].tolist()
    assert sum(p["set_hash"] for p in parts) % (1 << 64) == full["set_hash"]
    assert sum(p["paths_by_len"] for p in parts).tolist() == full["paths_by_len"].tolist()


def test_wide_class_chunked(ws):
    import torch
    g = I.gnp(2000, 0.005, I.GNP_SEED)
    # 256 pages of 1024 records (~69 MB) cannot hold the ~12 M-path F_6, so levels are split; a page
    # must still fit one page of children (fan-out up to ~8 here), see DESIGN.md §5
    small = torch.empty(256 * 1024 * 264, dtype=torch.uint8, device="cuda")
    got = binding.enumerate_cycles(*g, workspace=small, max_len=7, record_format=1)
    assert got["stats"]["chunks"] > got["stats"]["rounds"]
    assert_same(got, oracle.enumerate_cycles(*g, max_len=7, nthreads=NT))
    small = torch.empty(40 << 20, dtype=torch.uint8, device="cuda")  # F_6 alone is 430 MB of lists
    got = binding.enumerate_cycles(*g, workspace=small, max_len=8, record_format=2)
    assert got["stats"]["chunks"] > got["stats"]["rounds"]
    assert_same(got, oracle.enumerate_cycles(*g, max_len=8, nthreads=NT))


def test_repeat_runs_deterministic(ws):
    g = I.grid(6, 6)
    a = gpu(g, ws)
    for _ in range(3):
        assert_same(gpu(g, ws), a)


def test_stats_accounting(ws):
    """Frontier accounting: paths_expanded = sum |F_t|; with no length cap every
    path is written once and read once: paths_written = sum_t |F_t| and bytes_alg =
    record_bytes * (paths read + paths written by the expansions); t_dev > 0."""
    g = I.grid(6, 8)
    r = gpu(g, ws, profile=True)
    s = r["stats"]
    f = r["paths_by_len"]
    assert s["paths_expanded"] == int(f.sum())
    assert s["paths_written"] == int(f.sum()) and s["leaf_paths"] == 0
    written = int(f[4:].sum())  # every path of >= 4 vertices was written by an expansion
    assert s["bytes_alg"] == s["record_bytes"] * (int(f.sum()) + written)
    assert s["t_dev_ms"] > 0 and s["t_expand_ms"] > 0
    assert s["total_cycles"] == int(r["counts"].sum())


@pytest.mark.parametrize("name,g,K", [("grid6x8", I.grid(6, 8), 14), ("gnp100", I.gnp(100, 0.1, 4242), 8),
                                      ("gnp1200", I.gnp(1200, 0.006, 99), 8)])
def test_last_level_fusion_accounting(ws, name, g, K):
    """Count mode with max_len = K (last-level fusion): the paths of K-1 vertices
    are counted by the launch that creates them and never written; the counts, hash, |F_t| and
    candidates still equal the oracle's."""
    r = gpu(g, ws, max_len=K, profile=True)
    assert_same(r, oracle.enumerate_cycles(*g, max_len=K, nthreads=NT))
    s = r["stats"]
    f = r["paths_by_len"]
    assert s["leaf_paths"] == int(f[K - 1]) > 0
    assert s["paths_written"] == int(f[3:K - 1].sum())


def test_collect_mode_writes_every_path(ws):
    """Collect mode (S records) has no last-level fusion: every created path is written."""
    g = I.grid(5, 6)
    r = gpu(g, ws, collect=True, max_len=10)
    s = r["stats"]
    f = r["paths_by_len"]
    assert s["leaf_paths"] == 0
    assert s["paths_written"] == int(f.sum())


def test_k150_collect_at_scale(ws):
    """SURVEY §8(f)1, collect mode at the 10^8-cycle scale: K_{150,150} keeps all
    C(150,2)^2 = 124,880,625 cycles; cc_fetch_cycles streams them back in batches; every one is
    a 4-cycle <a, b, a', b'> alternating the two sides, no vertex set repeats, and the H-spec
    hash recomputed on the host from the fetched vertex lists equals the device's set hash."""
    g = I.complete_bipartite(150, 150)
    gr = binding.cc_graph_from_csr(*g)
    r = binding.cc_enumerate(gr, collect=True, workspace=ws)
    counts, h = binding.cc_count_by_length(r)
    total = math.comb(150, 2) ** 2
    assert int(counts[4]) == total and int(counts.sum()) == total
    assert binding.cc_num_stored_cycles(r) == total
    hs = 0
    codes = []
    batch = 1 << 24
    for first in range(0, total, batch):
        verts, offs = binding.cc_fetch_cycles(r, first, batch)
        k = len(offs) - 1
        assert np.all(np.diff(offs.astype(np.int64)) == 4)
        v = verts.reshape(k, 4).astype(np.int64)
        side = v >= 150
        assert np.all(side[:, 0] == side[:, 2]) and np.all(side[:, 1] == side[:, 3])
        assert np.all(side[:, 0] != side[:, 1])
        s = np.sort(v, axis=1)
        codes.append((s[:, 0] << 27) | (s[:, 1] << 18) | (s[:, 2] << 9) | s[:, 3])
        hs = (hs + brute.hspec_hash_np(verts, offs)) & brute.M64
    codes = np.concatenate(codes)
    assert len(np.unique(codes)) == total
    assert hs == h
    # ... and equals the oracle's set hash of the whole graph (tests/golden/oracle_k150.json)
    import json
    assert f"{h:#018x}" == json.load(open(os.path.join(GOLDEN, "oracle_k150.json")))["set_hash"]


GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
BIG = {
    "p8x8": (lambda: I.grid(8, 8), 0), "k150": (lambda: I.complete_bipartite(150, 150), 0),
    "grid8x10": (lambda: I.grid(8, 10), 0), "gnp2000_k9": (lambda: I.gnp(2000, 0.005, I.GNP_SEED), 9),
    "gnp2000_k10": (lambda: I.gnp(2000, 0.005, I.GNP_SEED), 10), "p10x10": (lambda: I.grid(10, 10), 0),
}


@pytest.mark.parametrize("name", sorted(BIG))
def test_full_size_against_oracle_golden(ws, name):
    """The BASELINE configs at full size, in the launch configuration bench.py times (a large
    arena, count mode): counts, set hash, |F_t| and candidates equal the oracle's, stored in
    tests/golden/oracle_<name>.json by tests/golden/make_oracle_big.py (oracle/ only)."""
    import json

    import torch
    path = os.path.join(GOLDEN, f"oracle_{name}.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated yet")
    want = json.load(open(path))
    build_g, K = BIG[name]
    assert want["max_len"] == K
    free, _ = torch.cuda.mem_get_info()
    big = torch.empty(int(free * 0.8), dtype=torch.uint8, device="cuda")
    got = binding.enumerate_cycles(*build_g(), workspace=big, max_len=K)
    del big
    assert {str(k): int(v) for k, v in enumerate(got["counts"]) if v} == want["counts"]
    assert f"{got['set_hash']:#018x}" == want["set_hash"]
    assert {str(k): int(v) for k, v in enumerate(got["paths_by_len"]) if v} == want["paths_by_len"]
    assert got["candidates"] == want["candidates"]


@pytest.mark.parametrize("name,g,K", [("grid5x6", I.grid(5, 6), 0), ("grid6x10", I.grid(6, 10), 0),
                                      ("k8x8", I.complete_bipartite(8, 8), 0), ("grid7x10_k14", I.grid(7, 10), 14),
                                      ("gnp90", I.gnp(90, 0.08, 5), 9), ("p4x4", I.grid(4, 4), 0)])
def test_small_frontier_path(ws, name, g, K):
    """The small-frontier fast path (one cooperative launch for the first levels)
    gives the oracle's counts, hash, |F_t| and candidates, and so does the paged path alone
    (CC_NO_SMALL); on the small grids it replaces the per-level launches."""
    want = oracle.enumerate_cycles(*g, max_len=K, nthreads=NT)
    got = gpu(g, ws, max_len=K)
    assert_same(got, want)
    os.environ["CC_NO_SMALL"] = "1"
    try:
        paged = gpu(g, ws, max_len=K)
    finally:
        del os.environ["CC_NO_SMALL"]
    assert_same(paged, want)
    if name in ("grid5x6", "p4x4"):
        assert got["stats"]["launches"] == 2 < paged["stats"]["launches"]


@pytest.mark.parametrize("name,g,K", [
    ("star600", I.star(600), 6),                 # wide class, Delta = 600: bitset only, no cycles
    ("cycle700", I.cycle(700), 0),               # wide class, one chordless cycle of 700 vertices
    ("complete40", I.complete(40), 0),           # triangles only: C(40, 3)
    ("gnp2015_list", I.gnp(2015, 0.0018, 77), 14),  # the largest n, the longest list records
    ("grid30x30_isolated", I.edges_to_csr(1000, [(a, b) for a, b in zip(*np.nonzero(np.triu(np.eye(900, k=1) + np.eye(900, k=30))))
                                                 if (b == a + 30) or (a % 30 != 29)]), 8),  # 100 isolated vertices
])
def test_degenerate_and_extreme_graphs(ws, name, g, K):
    got = gpu(g, ws, max_len=K)
    assert_same(got, oracle.enumerate_cycles(*g, max_len=K, nthreads=NT))
    if name == "cycle700":
        assert int(got["counts"][700]) == 1 and int(got["counts"].sum()) == 1
    if name == "complete40":
        assert int(got["counts"][3]) == math.comb(40, 3) and int(got["counts"].sum()) == math.comb(40, 3)


@pytest.mark.parametrize("W", [2, 3])
def test_shard_fallback_when_an_unsharded_level_does_not_fit(ws, W):
    """an unsharded level whose children overflow the arena is partitioned
    on the spot (shard_now).  Its child level must inherit the partition that the COMMITTED
    expansion used, so the shard sums still equal the whole.  A small arena and a huge
    min_shard_paths make every split happen through that fallback."""
    import torch
    g = I.grid(7, 8)
    small = torch.empty(160 * 1024 * 20, dtype=torch.uint8, device="cuda")
    full = oracle.enumerate_cycles(*g, nthreads=NT)
    parts = [binding.enumerate_cycles(*g, workspace=small, shard_index=i, shard_count=W,
                                      min_shard_paths=1 << 30) for i in range(W)]
    assert sum(p["counts"] for p in parts).tolist() == full["counts"].tolist()
    assert sum(p["set_hash"] for p in parts) % (1 << 64) == full["set_hash"]
    assert sum(p["paths_by_len"] for p in parts).tolist() == full["paths_by_len"].tolist()
    assert sum(p["candidates"] for p in parts) == full["candidates"]
    assert all(int(p["paths_by_len"].sum()) > 0 for p in parts)


@pytest.mark.parametrize("K", [1, 2])
def test_max_len_below_three_counts_nothing(ws, K):
    """a cap below 3 vertices admits no cycle, not even a triangle."""
    g = I.complete(6)
    got = gpu(g, ws, max_len=K)
    want = oracle.enumerate_cycles(*g, max_len=K)
    assert int(got["counts"].sum()) == 0 == int(want["counts"].sum())
    assert_same(got, want)


FUSED_GRAPHS = [("grid5x6", I.grid(5, 6), 0), ("grid6x7", I.grid(6, 7), 0), ("grid7x8", I.grid(7, 8), 0),
                ("grid7x10_k14", I.grid(7, 10), 14), ("grid7x10_k15", I.grid(7, 10), 15),
                ("grid6x10_k9", I.grid(6, 10), 9), ("p8x3", I.grid(8, 3), 0), ("c40", I.cycle(40), 0),
                ("grid6x6_k5", I.grid(6, 6), 5), ("grid6x6_k4", I.grid(6, 6), 4),
                # n = 104 / 105: the last packable two-word graph (8-bit ids) and the first unpacked
                ("grid8x13_k22", I.grid(8, 13), 22), ("grid7x15_k22", I.grid(7, 15), 22), ("c104", I.cycle(104), 0)]


@pytest.mark.parametrize("fq", ["1", "0"])
@pytest.mark.parametrize("name,g,K", FUSED_GRAPHS, ids=[x[0] for x in FUSED_GRAPHS])
def test_fused_two_level_kernel_every_level(ws, name, g, K, fq):
    """k_expand_fused (grid class, DESIGN.md §2 step 3d) on every level (CC_FUSED_MIN=1): two
    levels per launch, output chunks with empty slots, single-level and last-level-fusion
    launches near the cap.  Counts, hash, |F_t| and candidates equal the oracle's; the empty
    slots never count.  fq = 1: packed records take the full-round queue kernel k_expand_fq."""
    want = oracle.enumerate_cycles(*g, max_len=K, nthreads=NT)
    os.environ["CC_FUSED_MIN"] = "1"
    os.environ["CC_NO_SMALL"] = "1"
    os.environ["CC_FQ"] = fq
    try:
        got = gpu(g, ws, max_len=K)
    finally:
        del os.environ["CC_FUSED_MIN"]
        del os.environ["CC_NO_SMALL"]
        del os.environ["CC_FQ"]
    assert_same(got, want)
    s = got["stats"]
    f = got["paths_by_len"]
    # every level but the fused intermediates is written; levelsync counts each once read/written
    assert s["paths_expanded"] == int(f.sum())
    assert s["slots_moved"] >= s["bytes_alg"] // s["record_bytes"]


@pytest.mark.parametrize("name,g,rec", [("grid8x13", I.grid(8, 13), 24), ("grid7x15", I.grid(7, 15), 28)])
def test_packed_id_width_boundary(ws, name, g, rec):
    """Two-word records pack v1, v2, vt as 8-bit ids above bit n iff 128 - n >= 24 (n <= 104,
    cc::packed_id_bits); n = 105 keeps the ids in a separate u32 array.  Both equal the oracle."""
    want = oracle.enumerate_cycles(*g, max_len=20, nthreads=NT)
    got = gpu(g, ws, max_len=20)
    assert_same(got, want)
    assert got["stats"]["record_bytes"] == rec


@pytest.mark.parametrize("kb", [1024, 4096])
def test_fused_kernel_small_arena_chunks(ws, kb):
    """The fused kernel under the deepest-first chunk scheduler: a P7xP8 arena of 1 MB / 4 MB
    forces chunked, retried (overflowing) launches and sub-page chunks; results unchanged."""
    import torch
    g = I.grid(7, 8)
    small = torch.empty(kb * 1024, dtype=torch.uint8, device="cuda")
    os.environ["CC_FUSED_MIN"] = "1"
    try:
        got = binding.enumerate_cycles(*g, workspace=small)
        parts = [binding.enumerate_cycles(*g, workspace=small, shard_index=i, shard_count=2, min_shard_paths=64)
                 for i in range(2)]
    finally:
        del os.environ["CC_FUSED_MIN"]
    want = oracle.enumerate_cycles(*g, nthreads=NT)
    assert_same(got, want)
    assert got["stats"]["chunks"] > got["stats"]["rounds"] // 2
    assert sum(p["counts"] for p in parts).tolist() == want["counts"].tolist()
    assert sum(p["set_hash"] for p in parts) % (1 << 64) == want["set_hash"]
    assert sum(p["paths_by_len"] for p in parts).tolist() == want["paths_by_len"].tolist()


def _cycle_codes(verts, offs, n):
    """Per cycle: the vertex set as an n-bit mask (n <= 64) and a position-weighted hash of the
    canonical sequence -- to compare two cycle lists of 10^6 entries with numpy."""
    verts = np.asarray(verts, dtype=np.uint64)
    offs = np.asarray(offs, dtype=np.int64)
    k = len(offs) - 1
    cyc = np.repeat(np.arange(k), np.diff(offs))
    pos = np.arange(len(verts), dtype=np.int64) - offs[:-1][cyc]
    mask = np.bitwise_or.reduceat(np.left_shift(np.uint64(1), verts), offs[:-1])
    w = (verts + np.uint64(1)) * ((pos.astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15)) | np.uint64(1))
    seq = np.add.reduceat(w, offs[:-1])
    return mask, seq


def test_p8x8_collect_list_equals_oracle(ws):
    """P8xP8 in collect mode (1,743,247 cycles): the fetched cycle list equals the
    oracle's, as vertex sets and as canonical sequences (same labelling on both sides)."""
    import json
    g = I.grid(8, 8)
    gr = binding.cc_graph_from_csr(*g)
    r = binding.cc_enumerate(gr, collect=True, workspace=ws)
    counts, h = binding.cc_count_by_length(r)
    want = oracle.enumerate_cycles(*g, collect=True, raw=True, collect_cap=1 << 21)
    assert counts.tolist() == want["counts"].tolist() and h == want["set_hash"]
    assert f"{h:#018x}" == json.load(open(os.path.join(GOLDEN, "oracle_p8x8.json")))["set_hash"]
    verts, offs = binding.cc_fetch_cycles(r)
    gm, gs = _cycle_codes(verts, offs, 64)
    wm, wsq = _cycle_codes(want["vertices"], want["offsets"], 64)
    assert len(gm) == len(wm) == 1743247
    assert len(np.unique(gm)) == len(gm)  # exactly once
    assert np.array_equal(np.sort(gm), np.sort(wm))
    assert np.array_equal(np.sort(gs), np.sort(wsq))


CHAIN_GRAPHS = [("k100x100", I.complete_bipartite(100, 100), 0), ("gnp300", I.gnp(300, 0.03, 11), 8),
                ("grid12x12_k20", I.grid(12, 12), 20), ("grid12x12_k5", I.grid(12, 12), 5),
                ("grid12x12_k4", I.grid(12, 12), 4), ("k60x70_k3", I.complete_bipartite(60, 70), 3)]


@pytest.mark.parametrize("name,g,K", CHAIN_GRAPHS, ids=[x[0] for x in CHAIN_GRAPHS])
def test_stage1_chained_with_first_expansion(ws, name, g, K):
    """Stage 1 and the expansion of F_3 queued back to back with one host round trip (graphs
    outside the small-frontier path): same results as the unchained path and the oracle,
    including the last-level and no-children cases at level 3 (K = 5, 4, 3)."""
    want = oracle.enumerate_cycles(*g, max_len=K, nthreads=NT)
    got = gpu(g, ws, max_len=K)
    assert_same(got, want)
    os.environ["CC_NO_CHAIN"] = "1"
    try:
        plain = gpu(g, ws, max_len=K)
    finally:
        del os.environ["CC_NO_CHAIN"]
    assert_same(plain, want)
    assert got["stats"]["paths_written"] == plain["stats"]["paths_written"]


WIDE_COLLECT = [("gnp600_k7", I.gnp(600, 0.01, 5), 7), ("gnp2000_k6", I.gnp(2000, 0.005, I.GNP_SEED), 6),
                ("gnp2015_k14", I.gnp(2015, 0.0018, 77), 14), ("gnp700_k4", I.gnp(700, 0.008, 11), 4)]


@pytest.mark.parametrize("name,g,K", WIDE_COLLECT, ids=[x[0] for x in WIDE_COLLECT])
def test_wide_collect_list_equals_oracle(ws, name, g, K):
    """SURVEY §8(f)1 above n = 512: collect mode on vertex-list records (the list class) returns
    exactly the oracle's cycles as canonical sequences, including triangles from Stage 1 and the
    closures of the fused last level."""
    got = gpu(g, ws, max_len=K, collect=True)
    want = oracle.enumerate_cycles(*g, max_len=K, collect=True)
    assert_same(got, want)
    assert got["stats"]["record_format"] == 2
    assert len(got["cycles"]) == int(want["counts"].sum())
    assert sorted(map(tuple, got["cycles"])) == sorted(map(tuple, want["cycles"]))


def test_gnp2000_k9_collect_at_scale(ws):
    """G(2000, 0.005) at K = 9 in collect mode: 51,066,119 cycles stored on the device and fetched
    in batches; the H-spec hash recomputed on the host from the fetched lists equals the device
    hash and the oracle golden (tests/golden/oracle_gnp2000_k9.json)."""
    import json
    import torch
    want = json.load(open(os.path.join(GOLDEN, "oracle_gnp2000_k9.json")))
    g = I.gnp(2000, 0.005, I.GNP_SEED)
    free, _ = torch.cuda.mem_get_info()
    big = torch.empty(int(free * 0.6), dtype=torch.uint8, device="cuda")
    gr = binding.cc_graph_from_csr(*g)
    r = binding.cc_enumerate(gr, collect=True, workspace=big, max_len=9)
    counts, h = binding.cc_count_by_length(r)
    assert {str(k): int(v) for k, v in enumerate(counts) if v} == want["counts"]
    assert f"{h:#018x}" == want["set_hash"]
    total = want["total"]
    assert binding.cc_num_stored_cycles(r) == total
    hs = 0
    lens = np.zeros(10, dtype=np.int64)
    for first in range(0, total, 1 << 23):
        verts, offs = binding.cc_fetch_cycles(r, first, 1 << 23)
        lens += np.bincount(np.diff(offs.astype(np.int64)), minlength=10)[:10]
        hs = (hs + brute.hspec_hash_np(verts, offs)) & brute.M64
    assert hs == h
    assert {str(k): int(v) for k, v in enumerate(lens) if v} == want["counts"]
    del big
