"""CPU oracle for arXiv 1410.4876 chordless-cycle enumeration -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_1410_4876_b200``) never imports it, and it never imports the product path.

The arithmetic lives in ``oracle.c`` (plain C, compiled with gcc on first use); this module
only marshals arguments.  See the header of ``oracle.c`` for the paper passage each function
follows and DESIGN.md for the readings of the paper it takes.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

DEFAULT_SEED = 0x1410487600000000

ERRORS = {
    -1: "INVALID_ARGUMENT",
    -2: "INVALID_VERTEX",
    -3: "SELF_LOOP",
    -4: "NOT_SYMMETRIC",
    -5: "NO_MEMORY",
    -6: "BUFFER_TOO_SMALL",
}


class OracleError(RuntimeError):
    def __init__(self, code):
        self.code = code
        self.kind = ERRORS.get(code, str(code))
        super().__init__(f"oracle error {self.kind}")


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc -O2)."""
    with _lock:
        if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
            tmp = _LIB + f".tmp{os.getpid()}"
            subprocess.check_call(
                ["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-pthread", "-o", tmp, _SRC]
            )
            os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        lib.orc_mix.restype = ctypes.c_uint64
        lib.orc_mix.argtypes = [ctypes.c_uint64]
        lib.orc_validate.restype = ctypes.c_int
        lib.orc_validate.argtypes = [ctypes.c_int64, P, P]
        lib.orc_degree_labeling.restype = ctypes.c_int
        lib.orc_degree_labeling.argtypes = [ctypes.c_int64, P, P, P]
        lib.orc_triplets.restype = ctypes.c_int64
        lib.orc_triplets.argtypes = [ctypes.c_int64, P, P, P, P, ctypes.c_int64, P]
        lib.orc_enumerate.restype = ctypes.c_int
        lib.orc_enumerate.argtypes = [
            ctypes.c_int64, P, P, ctypes.c_uint32, ctypes.c_uint64, P, ctypes.c_int,
            ctypes.c_uint64, ctypes.c_uint64, P, P, P, P, P, ctypes.c_uint64, P,
            ctypes.c_uint64, P,
        ]
        lib.orc_enumerate_split.restype = ctypes.c_int
        lib.orc_enumerate_split.argtypes = [
            ctypes.c_int64, P, P, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, P, P, P, P,
        ]
        _lib = lib
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _csr(n, row_ptr, col):
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    return int(n), row_ptr, col


def mix(x: int) -> int:
    return int(_load().orc_mix(ctypes.c_uint64(x & 0xFFFFFFFFFFFFFFFF)))


def validate(n, row_ptr, col) -> str:
    n, row_ptr, col = _csr(n, row_ptr, col)
    rc = _load().orc_validate(n, _ptr(row_ptr), _ptr(col))
    return "OK" if rc == 0 else ERRORS.get(rc, str(rc))


def degree_labeling(n, row_ptr, col) -> np.ndarray:
    n, row_ptr, col = _csr(n, row_ptr, col)
    out = np.zeros(max(n, 1), dtype=np.int32)
    rc = _load().orc_degree_labeling(n, _ptr(row_ptr), _ptr(col), _ptr(out))
    if rc != 0:
        raise OracleError(rc)
    return out[:n]


def triplets(n, row_ptr, col, labels=None):
    """Returns (T as int32[|T|,3] rows (x,u,y), number of triangles)."""
    n, row_ptr, col = _csr(n, row_ptr, col)
    lab = None if labels is None else np.ascontiguousarray(labels, dtype=np.int32)
    ntri = np.zeros(1, dtype=np.uint64)
    lib = _load()
    nt = lib.orc_triplets(n, _ptr(row_ptr), _ptr(col), _ptr(lab), None, 0, _ptr(ntri))
    if nt < 0:
        raise OracleError(nt)
    out = np.zeros((max(nt, 1), 3), dtype=np.int32)
    lib.orc_triplets(n, _ptr(row_ptr), _ptr(col), _ptr(lab), _ptr(out), nt, _ptr(ntri))
    return out[:nt], int(ntri[0])


def enumerate_cycles(n, row_ptr, col, max_len: int = 0, seed: int = DEFAULT_SEED, labels=None,
                     nthreads: int = 1, collect: bool = False, root_stride: int = 1,
                     root_offset: int = 0, collect_cap: int = 1 << 20, raw: bool = False):
    """Run Alg. 1.  Returns a dict with

    counts (uint64[n+1], counts[k] = #chordless cycles with k vertices), set_hash,
    paths_by_len (uint64[n+1], paths of t vertices scanned), candidates, n_cycles and,
    if ``collect``, ``cycles``: list of canonical vertex sequences (original ids).
    """
    n, row_ptr, col = _csr(n, row_ptr, col)
    lab = None if labels is None else np.ascontiguousarray(labels, dtype=np.int32)
    counts = np.zeros(n + 1, dtype=np.uint64)
    pbl = np.zeros(n + 1, dtype=np.uint64)
    h = np.zeros(1, dtype=np.uint64)
    cand = np.zeros(1, dtype=np.uint64)
    ncyc = np.zeros(1, dtype=np.uint64)
    verts = offs = None
    vcap = ccap = 0
    if collect:
        ccap = collect_cap
        vcap = collect_cap * max(3, min(n, 32))
        verts = np.zeros(vcap, dtype=np.int32)
        offs = np.zeros(ccap + 1, dtype=np.uint64)
    rc = _load().orc_enumerate(
        n, _ptr(row_ptr), _ptr(col), max_len, seed, _ptr(lab), nthreads, root_stride,
        root_offset, _ptr(counts), _ptr(h), _ptr(pbl), _ptr(cand), _ptr(verts), vcap,
        _ptr(offs), ccap, _ptr(ncyc),
    )
    if rc == -6 and collect:
        return enumerate_cycles(n, row_ptr, col, max_len, seed, labels, nthreads, collect,
                                root_stride, root_offset,
                                collect_cap=max(2 * collect_cap, int(ncyc[0]) + 16), raw=raw)
    if rc != 0:
        raise OracleError(rc)
    out = dict(counts=counts, set_hash=int(h[0]), paths_by_len=pbl, candidates=int(cand[0]),
               n_cycles=int(ncyc[0]))
    if collect:
        k = int(ncyc[0])
        if raw:  # the same sequences as flat arrays (vertices, offsets[k + 1])
            out["vertices"], out["offsets"] = verts[:int(offs[k])], offs[:k + 1]
        else:
            out["cycles"] = [verts[int(offs[i]):int(offs[i + 1])].tolist() for i in range(k)]
    return out


def enumerate_cycles_split(n, row_ptr, col, max_len: int = 0, seed: int = DEFAULT_SEED,
                           nthreads: int = 1, split_len: int = 16):
    """Count mode of enumerate_cycles with a balanced multi-thread schedule for large runs
    (orc_enumerate_split): Alg. 1 down to paths of split_len vertices on one thread, then the
    subtrees of those paths on nthreads threads.  Same outputs as enumerate_cycles."""
    n, row_ptr, col = _csr(n, row_ptr, col)
    counts = np.zeros(n + 1, dtype=np.uint64)
    pbl = np.zeros(n + 1, dtype=np.uint64)
    h = np.zeros(1, dtype=np.uint64)
    cand = np.zeros(1, dtype=np.uint64)
    rc = _load().orc_enumerate_split(n, _ptr(row_ptr), _ptr(col), max_len, seed, nthreads, split_len,
                                     _ptr(counts), _ptr(h), _ptr(pbl), _ptr(cand))
    if rc != 0:
        raise OracleError(rc)
    return dict(counts=counts, set_hash=int(h[0]), paths_by_len=pbl, candidates=int(cand[0]))
