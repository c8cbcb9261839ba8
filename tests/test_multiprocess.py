"""N > 1 host path on CPU: two processes on the gloo backend combine per-shard results with the
same code bench.py uses (paper_1410_4876_b200.dist).  Each rank's shard result comes from the
oracle's root sample (rank r keeps roots with mix(x<<42|u<<21|y) % W == r), so the combined
counts / hash / path count must equal the oracle's unsharded run exactly."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, graph_name, out_q):
    import torch.distributed as dist

    import oracle
    from paper_1410_4876_b200 import dist as D, inputs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = inputs.named(graph_name)
    r = oracle.enumerate_cycles(*g, root_stride=world, root_offset=rank)
    counts, h, paths = D.combine_shards(r["counts"], r["set_hash"], int(r["paths_by_len"].sum()))
    t = D.max_over_ranks(float(rank + 1))
    pr = D.gather_per_rank([float(rank + 1), float(int(r["paths_by_len"].sum()))])
    if rank == 0:
        out_q.put((counts.tolist(), h, paths, t, pr))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("graph_name", ["grid6x6", "k12x9"])
def test_gloo_combine_equals_unsharded(world, graph_name):
    import oracle
    from paper_1410_4876_b200 import inputs

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, graph_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    counts, h, paths, t, pr = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = oracle.enumerate_cycles(*inputs.named(graph_name))
    assert counts == full["counts"].tolist()
    assert h == full["set_hash"]
    assert paths == int(full["paths_by_len"].sum())
    assert t == float(world)
    # per-rank report (bench.py "per_rank"): every rank's row, in rank order, summing to the whole
    assert [row[0] for row in pr] == [float(r + 1) for r in range(world)]
    assert sum(row[1] for row in pr) == paths


def test_hash_wraps_mod_2_64():
    from paper_1410_4876_b200.dist import _i64_to_u64, _u64_to_i64
    for x in (0, 1, 2**63 - 1, 2**63, 2**64 - 1, 0x643A7125E816E7A1):
        assert _i64_to_u64(_u64_to_i64(x)) == x
    a, b = 0xF000000000000000, 0x2000000000000001
    s = (_u64_to_i64(a) + _u64_to_i64(b) + 2**63) % 2**64 - 2**63  # int64 wrap
    assert _i64_to_u64(s) == (a + b) % 2**64
