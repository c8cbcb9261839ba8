"""C-ABI checks that need no GPU: the library loads, exports every symbol include/*.h declares,
validates CSR input with the documented error kinds, computes the same degree labelling as the
oracle (host preprocessing), and fails loudly (no CPU fallback) without a GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
from paper_1410_4876_b200 import binding, build, inputs as I

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    build.build()
    return binding.load()


def _declared_functions():
    names = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            src = open(os.path.join(ROOT, "include", fn)).read()
            src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
            names |= set(re.findall(r"\b(cc_[a-z_]+)\s*\(", src))
    return names


def test_library_exports_every_declared_symbol(lib):
    declared = _declared_functions()
    assert declared, "no declarations parsed"
    assert declared == set(binding.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name


def test_struct_sizes_match_header(lib):
    o = binding.cc_options()
    lib.cc_options_init(ctypes.byref(o))
    assert o.struct_size == ctypes.sizeof(binding.cc_options)
    assert o.shard_count == 1 and o.device == -1


def test_version_names_sm100a(lib):
    assert "sm_100a" in binding.cc_version()


@pytest.mark.parametrize("name,g", [("p4x4", I.grid(4, 4)), ("k150", I.complete_bipartite(150, 150)),
                                    ("p10x10", I.grid(10, 10)), ("gnp", I.gnp(300, 0.05, 1)),
                                    ("wheel", I.wheel(100)), ("tree", I.random_tree(50, 2))])
def test_host_degree_labelling_equals_oracle(lib, name, g):
    """Both sides implement PAPER.md:53 with lowest-id ties (reading G1) independently:
    the library with an ordered set, the oracle with an O(n^2) scan."""
    gr = binding.cc_graph_from_csr(*g)
    assert binding.cc_graph_labels(gr).tolist() == oracle.degree_labeling(*g).tolist()
    n, m, d = binding.cc_graph_info(gr)
    assert (n, m, d) == (g[0], len(g[2]) // 2, int(np.diff(g[1]).max()))


def test_csr_validation_error_kinds(lib):
    rp = np.array([0, 1, 2], dtype=np.int64)
    binding.cc_graph_from_csr(2, rp, np.array([1, 0], dtype=np.int32))
    cases = [
        (2, rp, np.array([2, 0], dtype=np.int32), "CC_ERR_INVALID_VERTEX"),
        (2, rp, np.array([-1, 0], dtype=np.int32), "CC_ERR_INVALID_VERTEX"),
        (2, rp, np.array([0, 0], dtype=np.int32), "CC_ERR_SELF_LOOP"),
        (3, np.array([0, 1, 1, 1]), np.array([1], dtype=np.int32), "CC_ERR_NOT_SYMMETRIC"),
        (2, np.array([0, 2, 1]), np.array([1, 0], dtype=np.int32), "CC_ERR_INVALID_ARGUMENT"),
        (2, np.array([1, 2, 2]), np.array([1, 0], dtype=np.int32), "CC_ERR_INVALID_ARGUMENT"),
        (-1, np.array([0]), np.array([0], dtype=np.int32), "CC_ERR_INVALID_ARGUMENT"),
    ]
    for n, rp_, col, kind in cases:
        with pytest.raises(binding.CCError) as ei:
            binding.cc_graph_from_csr(n, rp_, col)
        assert ei.value.kind == kind
        assert binding.load().cc_last_error().decode()
    # duplicates merge, rows may be unsorted
    gr = binding.cc_graph_from_csr(3, np.array([0, 3, 5, 7]), np.array([2, 1, 2, 0, 2, 1, 0], dtype=np.int32))
    assert binding.cc_graph_info(gr) == (3, 3, 2)


def test_empty_and_tiny_graphs_build(lib):
    for n in range(0, 4):
        gr = binding.cc_graph_from_csr(n, np.zeros(n + 1, dtype=np.int64), np.zeros(0, dtype=np.int32))
        assert binding.cc_graph_info(gr) == (n, 0, 0)


def test_no_cpu_fallback_without_gpu(lib):
    """On a machine without a CUDA device cc_enumerate must fail, not silently compute."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    gr = binding.cc_graph_from_csr(*I.grid(4, 4))
    with pytest.raises(binding.CCError) as ei:
        binding.cc_enumerate(gr)
    assert ei.value.kind in ("CC_ERR_NO_DEVICE", "CC_ERR_CUDA")


def test_buffer_too_small_and_null_handles(lib):
    assert lib.cc_count_by_length(None, None, 0, None, None) == 1
    assert lib.cc_graph_info(None, None, None, None) == 1
    lib.cc_graph_free(None)
    lib.cc_result_free(None)
    assert lib.cc_status_string(5) == b"CC_ERR_CAPACITY"
