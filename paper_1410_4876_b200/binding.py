"""Thin ctypes binding of the C ABI in include/chordless.h (argument marshalling only).

Every step of the enumeration runs inside libchordless.so (host labelling + sm_100a kernels).
There is no fallback: if the library is missing or no GPU is present, the calls raise.
PyTorch is used only to supply device memory (the frontier workspace) and the CUDA stream.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# CC_LIBCHORDLESS overrides the library path (A/B builds of the same ABI)
LIB_PATH = os.environ.get("CC_LIBCHORDLESS") or os.path.join(HERE, "libchordless.so")

CC_STATUS = {
    0: "CC_OK", 1: "CC_ERR_INVALID_ARGUMENT", 2: "CC_ERR_INVALID_VERTEX", 3: "CC_ERR_SELF_LOOP",
    4: "CC_ERR_NOT_SYMMETRIC", 5: "CC_ERR_CAPACITY", 6: "CC_ERR_CUDA", 7: "CC_ERR_NOT_COLLECTED",
    8: "CC_ERR_BUFFER_TOO_SMALL", 9: "CC_ERR_TOO_LARGE", 10: "CC_ERR_NO_DEVICE",
}

# Every function include/chordless.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "cc_options_init", "cc_graph_from_csr", "cc_graph_free", "cc_graph_info", "cc_graph_labels",
    "cc_enumerate", "cc_count_by_length", "cc_paths_by_length", "cc_fetch_cycles",
    "cc_num_stored_cycles", "cc_result_stats", "cc_result_free", "cc_last_error",
    "cc_status_string", "cc_version",
]


class CCError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        self.kind = CC_STATUS.get(status, str(status))
        super().__init__(f"{self.kind}: {msg}")


class cc_options(ctypes.Structure):
    _fields_ = [
        ("struct_size", ctypes.c_uint32), ("device", ctypes.c_int32), ("stream", ctypes.c_void_p),
        ("max_len", ctypes.c_uint32), ("collect", ctypes.c_uint32), ("shard_index", ctypes.c_uint32),
        ("shard_count", ctypes.c_uint32), ("root_stride", ctypes.c_uint64),
        ("root_offset", ctypes.c_uint64), ("hash_seed", ctypes.c_uint64),
        ("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_uint64),
        ("collect_capacity", ctypes.c_uint64), ("profile", ctypes.c_uint32),
        ("min_shard_paths", ctypes.c_uint32), ("record_format", ctypes.c_uint32),
    ]


class cc_stats(ctypes.Structure):
    _fields_ = [
        ("struct_size", ctypes.c_uint32), ("n_words", ctypes.c_uint32),
        ("total_cycles", ctypes.c_uint64), ("paths_expanded", ctypes.c_uint64),
        ("candidates", ctypes.c_uint64), ("triplets", ctypes.c_uint64),
        ("stage1_pairs", ctypes.c_uint64), ("rounds", ctypes.c_uint64),
        ("launches", ctypes.c_uint64), ("chunks", ctypes.c_uint64),
        ("peak_arena_records", ctypes.c_uint64), ("arena_capacity", ctypes.c_uint64),
        ("record_bytes", ctypes.c_uint64), ("bytes_alg", ctypes.c_uint64),
        ("cycles_stored", ctypes.c_uint64), ("h2d_bytes", ctypes.c_uint64),
        ("d2h_bytes", ctypes.c_uint64), ("t_dev_ms", ctypes.c_double),
        ("t_expand_ms", ctypes.c_double), ("t_stage1_ms", ctypes.c_double),
        ("t_labeling_ms", ctypes.c_double), ("t_wall_ms", ctypes.c_double),
        ("leaf_paths", ctypes.c_uint64), ("paths_written", ctypes.c_uint64),
        ("record_format", ctypes.c_uint64), ("records_levelsync", ctypes.c_uint64),
        ("slots_moved", ctypes.c_uint64),
    ]


_lib = None


def load(path: str = LIB_PATH):
    """Load libchordless.so and declare the prototypes.  Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    lib = ctypes.CDLL(path)
    P, u64, i64, i32, sz = (ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32,
                            ctypes.c_size_t)
    st = ctypes.c_int
    lib.cc_options_init.restype = None
    lib.cc_options_init.argtypes = [ctypes.POINTER(cc_options)]
    lib.cc_graph_from_csr.restype = st
    lib.cc_graph_from_csr.argtypes = [i64, P, P, ctypes.POINTER(P)]
    lib.cc_graph_free.restype = None
    lib.cc_graph_free.argtypes = [P]
    lib.cc_graph_info.restype = st
    lib.cc_graph_info.argtypes = [P, P, P, P]
    lib.cc_graph_labels.restype = st
    lib.cc_graph_labels.argtypes = [P, P]
    lib.cc_enumerate.restype = st
    lib.cc_enumerate.argtypes = [P, ctypes.POINTER(cc_options), ctypes.POINTER(P)]
    lib.cc_count_by_length.restype = st
    lib.cc_count_by_length.argtypes = [P, P, sz, P, P]
    lib.cc_paths_by_length.restype = st
    lib.cc_paths_by_length.argtypes = [P, P, sz, P]
    lib.cc_fetch_cycles.restype = st
    lib.cc_fetch_cycles.argtypes = [P, u64, u64, P, sz, P, P]
    lib.cc_num_stored_cycles.restype = st
    lib.cc_num_stored_cycles.argtypes = [P, P]
    lib.cc_result_stats.restype = st
    lib.cc_result_stats.argtypes = [P, ctypes.POINTER(cc_stats)]
    lib.cc_result_free.restype = None
    lib.cc_result_free.argtypes = [P]
    lib.cc_last_error.restype = ctypes.c_char_p
    lib.cc_last_error.argtypes = []
    lib.cc_status_string.restype = ctypes.c_char_p
    lib.cc_status_string.argtypes = [st]
    lib.cc_version.restype = ctypes.c_char_p
    lib.cc_version.argtypes = []
    _lib = lib
    return lib


def _check(status: int):
    if status != 0:
        raise CCError(status, load().cc_last_error().decode())


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class Graph:
    """Owns a cc_graph*.  Built from host CSR (copied)."""

    def __init__(self, handle):
        self._h = handle

    @property
    def handle(self):
        return self._h

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.cc_graph_free(self._h)
            self._h = None


class Result:
    """Owns a cc_result*."""

    def __init__(self, handle, n: int):
        self._h = handle
        self.n = n

    @property
    def handle(self):
        return self._h

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.cc_result_free(self._h)
            self._h = None


def cc_graph_from_csr(n: int, row_ptr, col_idx) -> Graph:
    lib = load()
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    if ci.size == 0:
        ci = np.zeros(1, dtype=np.int32)
    h = ctypes.c_void_p()
    _check(lib.cc_graph_from_csr(int(n), _ptr(rp), _ptr(ci), ctypes.byref(h)))
    return Graph(h)


def cc_graph_info(g: Graph):
    n, m, d = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _check(load().cc_graph_info(g.handle, ctypes.byref(n), ctypes.byref(m), ctypes.byref(d)))
    return n.value, m.value, d.value


def cc_graph_labels(g: Graph) -> np.ndarray:
    n, _, _ = cc_graph_info(g)
    lab = np.zeros(max(n, 1), dtype=np.int32)
    _check(load().cc_graph_labels(g.handle, _ptr(lab)))
    return lab[:n]


def make_options(device: int = -1, stream=None, max_len: int = 0, collect: bool = False,
                 shard_index: int = 0, shard_count: int = 1, root_stride: int = 0,
                 root_offset: int = 0, hash_seed: int = 0, workspace=None, workspace_bytes: int = 0,
                 collect_capacity: int = 0, profile: bool = False, min_shard_paths: int = 0,
                 record_format: int = 0):
    o = cc_options()
    load().cc_options_init(ctypes.byref(o))
    o.device = device
    o.stream = stream
    o.max_len = max_len
    o.collect = 1 if collect else 0
    o.shard_index = shard_index
    o.shard_count = shard_count
    o.root_stride = root_stride
    o.root_offset = root_offset
    o.hash_seed = hash_seed
    if workspace is not None:
        # a torch tensor (device memory owned by the caller) or a raw (pointer, bytes) pair
        if isinstance(workspace, tuple):
            o.workspace, o.workspace_bytes = workspace
        else:
            o.workspace = workspace.data_ptr()
            o.workspace_bytes = workspace.numel() * workspace.element_size()
    else:
        o.workspace_bytes = workspace_bytes
    o.collect_capacity = collect_capacity
    o.profile = 1 if profile else 0
    o.min_shard_paths = min_shard_paths
    o.record_format = record_format
    return o


def cc_enumerate(g: Graph, opts: cc_options | None = None, **kw) -> Result:
    if opts is None:
        opts = make_options(**kw)
    h = ctypes.c_void_p()
    _check(load().cc_enumerate(g.handle, ctypes.byref(opts), ctypes.byref(h)))
    n, _, _ = cc_graph_info(g)
    return Result(h, n)


def cc_count_by_length(r: Result):
    lib = load()
    nl = ctypes.c_size_t()
    hs = ctypes.c_uint64()
    _check(lib.cc_count_by_length(r.handle, None, 0, ctypes.byref(nl), ctypes.byref(hs)))
    counts = np.zeros(max(nl.value, 1), dtype=np.uint64)
    _check(lib.cc_count_by_length(r.handle, _ptr(counts), counts.size, ctypes.byref(nl),
                                  ctypes.byref(hs)))
    return counts[:nl.value], int(hs.value)


def cc_paths_by_length(r: Result) -> np.ndarray:
    lib = load()
    nl = ctypes.c_size_t()
    _check(lib.cc_paths_by_length(r.handle, None, 0, ctypes.byref(nl)))
    paths = np.zeros(max(nl.value, 1), dtype=np.uint64)
    _check(lib.cc_paths_by_length(r.handle, _ptr(paths), paths.size, ctypes.byref(nl)))
    return paths[:nl.value]


def cc_num_stored_cycles(r: Result) -> int:
    k = ctypes.c_uint64()
    _check(load().cc_num_stored_cycles(r.handle, ctypes.byref(k)))
    return int(k.value)


def cc_fetch_cycles(r: Result, first: int = 0, max_cycles: int | None = None, max_len: int | None = None):
    """Returns (vertices int32[], offsets uint64[k+1]) for cycles [first, first+k).

    The vertex buffer is sized from the longest stored cycle (``max_len``, default: the
    largest k with counts[k] > 0), so one library call fetches the batch; the two-call sizing
    protocol of the C ABI is the fallback."""
    lib = load()
    total = cc_num_stored_cycles(r)
    if max_cycles is None:
        max_cycles = max(total - first, 0)
    k = min(max_cycles, max(total - first, 0))
    if max_len is None:
        counts, _ = cc_count_by_length(r)
        nz = np.nonzero(counts)[0]
        max_len = int(nz[-1]) if len(nz) else 0
    offsets = np.empty(max_cycles + 1, dtype=np.uint64)
    verts = np.empty(max(k * max_len, 1), dtype=np.int32)
    nf = ctypes.c_uint64()
    st = lib.cc_fetch_cycles(r.handle, first, max_cycles, _ptr(verts), verts.size, _ptr(offsets),
                             ctypes.byref(nf))
    if st == 8:  # BUFFER_TOO_SMALL (max_len underestimated): offsets tell the size
        verts = np.empty(max(int(offsets[k]), 1), dtype=np.int32)
        st = lib.cc_fetch_cycles(r.handle, first, max_cycles, _ptr(verts), verts.size, _ptr(offsets),
                                 ctypes.byref(nf))
    _check(st)
    k = int(nf.value)
    if k == 0:
        offsets[0] = 0
    return verts[:int(offsets[k])], offsets[:k + 1]


def cc_result_stats(r: Result) -> dict:
    s = cc_stats()
    s.struct_size = ctypes.sizeof(cc_stats)
    _check(load().cc_result_stats(r.handle, ctypes.byref(s)))
    return {name: getattr(s, name) for name, _ in cc_stats._fields_}


def cc_version() -> str:
    return load().cc_version().decode()


# ---------------------------------------------------------------------------- convenience
def enumerate_cycles(n, row_ptr, col, *, collect: bool = False, workspace=None, stream=None,
                     **kw) -> dict:
    """cc_graph_from_csr + cc_enumerate + cc_count_by_length (+ cc_fetch_cycles).

    ``stream`` defaults to torch's current stream on the current device when torch is
    importable; ``workspace`` may be a torch uint8 CUDA tensor (else the library allocates).
    """
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                stream = torch.cuda.current_stream().cuda_stream
        except ImportError:
            pass
    g = cc_graph_from_csr(n, row_ptr, col)
    r = cc_enumerate(g, collect=collect, workspace=workspace, stream=stream, **kw)
    counts, h = cc_count_by_length(r)
    out = dict(counts=counts, set_hash=h, paths_by_len=cc_paths_by_length(r),
               stats=cc_result_stats(r), labels=cc_graph_labels(g))
    out["candidates"] = out["stats"]["candidates"]
    if collect:
        verts, offs = cc_fetch_cycles(r)
        out["cycles"] = [verts[int(offs[i]):int(offs[i + 1])].tolist() for i in range(len(offs) - 1)]
    return out
