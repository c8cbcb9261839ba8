"""Write tests/golden/oracle_<name>.json from the CPU oracle ONLY (no CUDA path involved).

    python tests/golden/make_oracle_big.py p10x10 [--threads N]

Each file holds the oracle's per-length counts, set hash, |F_t| per t, candidates, and the
wall time and thread count of the run.  These are the expected values of the full-size GPU
parity tests for workloads too large to run the oracle inside the test suite.
"""
import argparse
import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1410_4876_b200 import inputs  # noqa: E402

CONFIGS = {
    "p10x10": dict(graph=lambda: inputs.grid(10, 10), max_len=0, split_len=18),
    "grid8x10": dict(graph=lambda: inputs.grid(8, 10), max_len=0, split_len=16),
    "grid9x9": dict(graph=lambda: inputs.grid(9, 9), max_len=0, split_len=16),
    "gnp2000_k8": dict(graph=lambda: inputs.gnp(2000, 0.005, inputs.GNP_SEED), max_len=8),
    "gnp2000_k9": dict(graph=lambda: inputs.gnp(2000, 0.005, inputs.GNP_SEED), max_len=9),
    "gnp2000_k10": dict(graph=lambda: inputs.gnp(2000, 0.005, inputs.GNP_SEED), max_len=10),
    "k150": dict(graph=lambda: inputs.complete_bipartite(150, 150), max_len=0),
    "p8x8": dict(graph=lambda: inputs.grid(8, 8), max_len=0, split_len=12),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name", choices=sorted(CONFIGS))
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    a = ap.parse_args()
    cfg = CONFIGS[a.name]
    g = cfg["graph"]()
    t0 = time.time()
    # balanced schedule (orc_enumerate_split, pinned equal to orc_enumerate by
    # tests/test_oracle_pins.py::test_split_driver_equals_sequential_oracle)
    r = oracle.enumerate_cycles_split(*g, max_len=cfg["max_len"], nthreads=a.threads,
                                      split_len=cfg.get("split_len", 8))
    dt = time.time() - t0
    out = {
        "name": a.name, "n": g[0], "m": len(g[2]) // 2, "max_len": cfg["max_len"],
        "counts": {str(k): int(v) for k, v in enumerate(r["counts"]) if v},
        "total": int(r["counts"].sum()), "set_hash": f"{r['set_hash']:#018x}",
        "paths_by_len": {str(k): int(v) for k, v in enumerate(r["paths_by_len"]) if v},
        "paths_total": int(r["paths_by_len"].sum()), "candidates": r["candidates"],
        "oracle_seconds": dt, "oracle_threads": a.threads, "split_len": cfg.get("split_len", 8),
        "generated_by": "tests/golden/make_oracle_big.py (oracle/ only)",
        # the input graph itself, so a change of the generator (e.g. numpy's PCG64 stream) is
        # caught as a different graph rather than as a wrong count
        "csr_sha256": hashlib.sha256(g[1].astype("<i8").tobytes() + g[2].astype("<i4").tobytes()).hexdigest(),
    }
    with open(os.path.join(HERE, f"oracle_{a.name}.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: out[k] for k in ("name", "total", "set_hash", "paths_total", "oracle_seconds")}))


if __name__ == "__main__":
    main()
