"""Per-shard work of the multi-GPU partition, measured on ONE GPU (shards run one after another).

    python tools/shard_balance.py p10x10 --shards 2 4 8 --min-shard-paths 0 65536

For each (W, min_shard_paths) it runs cc_enumerate(shard_index=i, shard_count=W) for every i and
prints one JSON line: paths and device ms per shard, max/mean imbalance of both, and the check
that the shard sums equal the unsharded counts + hash.  A W-GPU run takes max_i t_i, so
max/mean of the device time is the strong-scaling loss the static partition causes.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1410_4876_b200 import binding, inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload")
ap.add_argument("--shards", type=int, nargs="+", default=[2, 4, 8])
ap.add_argument("--min-shard-paths", type=int, nargs="+", default=[0])
ap.add_argument("--max-len", type=int, default=0)
a = ap.parse_args()

g = inputs.named(a.workload)
free, _ = torch.cuda.mem_get_info()
ws = torch.empty(int(free * 0.85) - (1 << 30), dtype=torch.uint8, device="cuda")
gr = binding.cc_graph_from_csr(*g)
stream = torch.cuda.current_stream().cuda_stream


def run(i, w, msp):
    r = binding.cc_enumerate(gr, workspace=ws, max_len=a.max_len, stream=stream, shard_index=i,
                             shard_count=w, min_shard_paths=msp)
    c, h = binding.cc_count_by_length(r)
    s = binding.cc_result_stats(r)
    return c.astype(np.uint64), h, s


c0, h0, s0 = run(0, 1, 0)
c0, h0, s0 = run(0, 1, 0)  # warm
print(json.dumps({"workload": a.workload, "W": 1, "cycles": int(c0.sum()), "paths": s0["paths_expanded"],
                  "t_dev_ms": s0["t_dev_ms"]}), flush=True)
for w in a.shards:
    for msp in a.min_shard_paths:
        tot = np.zeros_like(c0)
        hs = 0
        paths, ms = [], []
        for i in range(w):
            c, h, s = run(i, w, msp)
            n = min(len(tot), len(c))
            tot[:n] += c[:n]
            hs = (hs + h) & ((1 << 64) - 1)
            paths.append(int(s["paths_expanded"]))
            ms.append(float(s["t_dev_ms"]))
        print(json.dumps({
            "workload": a.workload, "W": w, "min_shard_paths": msp or "default",
            "exact": bool((tot == c0).all() and hs == h0),
            "paths": paths, "t_dev_ms": [round(x, 2) for x in ms],
            "paths_max_over_mean": max(paths) / (sum(paths) / w),
            "time_max_over_mean": max(ms) / (sum(ms) / w),
            "ideal_speedup_vs_W1": s0["t_dev_ms"] / max(ms),
        }), flush=True)
