"""Run one enumeration of a named workload through the C ABI (for ncu / nsight captures).

    python tools/run_once.py p10x10 [--max-len K] [--repeat R] [--workspace-gb G]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1410_4876_b200 import binding, inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload")
ap.add_argument("--max-len", type=int, default=0)
ap.add_argument("--repeat", type=int, default=1)
ap.add_argument("--workspace-gb", type=float, default=0)
ap.add_argument("--profile", action="store_true")
ap.add_argument("--collect", action="store_true", help="collect mode; also time cc_fetch_cycles of every cycle")
ap.add_argument("--collect-capacity", type=int, default=0)
a = ap.parse_args()
g = inputs.named(a.workload)
free, _ = torch.cuda.mem_get_info()
wsb = int(a.workspace_gb * (1 << 30)) if a.workspace_gb else int(free * 0.85) - (1 << 30)
ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
gr = binding.cc_graph_from_csr(*g)
for i in range(a.repeat):
    t0 = time.perf_counter()
    r = binding.cc_enumerate(gr, workspace=ws, max_len=a.max_len, stream=torch.cuda.current_stream().cuda_stream,
                             profile=a.profile, collect=a.collect, collect_capacity=a.collect_capacity)
    dt = time.perf_counter() - t0
    c, h = binding.cc_count_by_length(r)
    s = binding.cc_result_stats(r)
    out = {"workload": a.workload, "wall_s": dt, "cycles": int(c.sum()), "hash": f"{h:#018x}",
           "paths": s["paths_expanded"], "launches": s["launches"], "t_dev_ms": s["t_dev_ms"],
           "t_expand_ms": s["t_expand_ms"], "peak": s["peak_arena_records"], "cap": s["arena_capacity"]}
    if a.collect:
        t1 = time.perf_counter()
        k = binding.cc_num_stored_cycles(r)
        nv = 0
        for first in range(0, k, 1 << 24):
            verts, offs = binding.cc_fetch_cycles(r, first, 1 << 24)
            nv += len(verts)
        out.update(stored=k, fetch_s=time.perf_counter() - t1, fetched_vertices=nv)
    print(json.dumps(out), flush=True)
