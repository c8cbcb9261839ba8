"""Multi-GPU combine of per-shard results.

Each rank enumerates its shard through the C ABI (``cc_options.shard_index/shard_count``); the
only data-path exchange is ONE all_reduce(SUM) of an int64 vector [counts[0..n], set_hash,
paths] plus a MAX of the device time.  The set hash is a sum mod 2^64 (H-spec), so it travels
as the int64 with the same bits: two's-complement addition wraps exactly like uint64 addition.
Works on NCCL (CUDA tensors, NVLink) and on gloo (CPU tensors, for the CPU tests).
"""
from __future__ import annotations

import numpy as np


def _u64_to_i64(x: int) -> int:
    return int(np.array([x & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64).view(np.int64)[0])


def _i64_to_u64(x: int) -> int:
    return int(np.array([x], dtype=np.int64).view(np.uint64)[0])


def combine_shards(counts, set_hash: int, paths: int, device=None, group=None):
    """Sum per-length counts, the set hash (mod 2^64) and the path count over all ranks."""
    import torch
    import torch.distributed as dist

    counts = np.asarray(counts, dtype=np.uint64)
    v = np.concatenate([counts.astype(np.int64), np.array([_u64_to_i64(set_hash), int(paths)], dtype=np.int64)])
    t = torch.from_numpy(v)
    if device is not None:
        t = t.to(device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    v = t.cpu().numpy()
    return v[:-2].astype(np.uint64), _i64_to_u64(int(v[-2])), int(v[-1])


def max_over_ranks(x: float, device=None, group=None) -> float:
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(x)], dtype=torch.float64)
    if device is not None:
        t = t.to(device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def min_over_ranks(x: float, device=None, group=None) -> float:
    """MIN of a scalar (e.g. the arena size every rank must share, include/chordless.h)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(x)], dtype=torch.float64)
    if device is not None:
        t = t.to(device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return float(t.item())


def gather_per_rank(values, device=None, group=None):
    """All ranks' small float vectors (e.g. [device ms, paths]) for the imbalance report,
    SURVEY §8(e) -- reporting only, not on the data path."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(v) for v in values], dtype=torch.float64)
    if device is not None:
        t = t.to(device)
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, t, group=group)
    return [[float(x) for x in o.cpu().tolist()] for o in out]
