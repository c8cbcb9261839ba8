"""N > 1 on the GPU path: W processes (one per shard, all on the leased GPU, gloo for the two
small reductions) each run the real cc_enumerate on their shard through the C ABI, and
paper_1410_4876_b200.dist.combine_shards -- the code bench.py uses -- sums them.  The combined
counts, set hash and path count must equal the oracle's full-size goldens (tests/golden/).
SURVEY §8(e): the only data exchange is one all_reduce(SUM) of counts + hash + paths."""
import json
import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = {"p8x8": ("grid8x8", 0), "gnp2000_k9": ("gnp2000", 9)}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, graph_name, max_len, ws_bytes, out_q):
    import torch
    import torch.distributed as dist

    from paper_1410_4876_b200 import binding, dist as D, inputs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda:0")
    g = inputs.named(graph_name)
    # min_shard_paths 2^16: P8x8 (peak level 2.9e6 paths) is split at every W tested
    r = binding.enumerate_cycles(*g, workspace=ws, max_len=max_len, shard_index=rank, shard_count=world,
                                 min_shard_paths=1 << 16)
    counts, h, paths = D.combine_shards(r["counts"], r["set_hash"], int(r["paths_by_len"].sum()))
    _, _, cand = D.combine_shards(r["counts"][:1] * 0, 0, int(r["candidates"]))
    mine = int(r["paths_by_len"].sum())
    if rank == 0:
        out_q.put((counts.tolist(), h, paths, cand, mine))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", sorted(CASES))
def test_processes_shard_and_combine_to_the_golden(world, name):
    want = json.load(open(os.path.join(GOLDEN, f"oracle_{name}.json")))
    graph_name, K = CASES[name]
    assert want["max_len"] == K
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, graph_name, K, 8 << 30, q)) for r in range(world)]
    for p in procs:
        p.start()
    counts, h, paths, cand, mine = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert {str(k): int(v) for k, v in enumerate(counts) if v} == want["counts"]
    assert f"{h:#018x}" == want["set_hash"]
    assert paths == want["paths_total"]
    assert cand == want["candidates"]
    assert 0 < mine < paths  # rank 0 did a real share, not everything
