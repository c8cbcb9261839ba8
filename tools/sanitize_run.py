"""Small enumerations through every kernel class, for compute-sanitizer runs:
    compute-sanitizer --tool memcheck python tools/sanitize_run.py
Exits non-zero if any result differs from the oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1410_4876_b200 import binding, inputs as I  # noqa: E402

ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
cases = [
    ("p6x6 count (B-mode, Delta<=4 kernel)", I.grid(6, 6), {}),
    ("p5x5 collect (S-mode thread kernel)", I.grid(5, 5), dict(collect=True)),
    ("k12x12 count (B-mode, Delta>4)", I.complete_bipartite(12, 12), {}),
    ("k40x40 collect (S-mode warp kernel)", I.complete_bipartite(40, 40), dict(collect=True)),
    ("gnp200 count shard 1/3 (filter kernel)", I.gnp(200, 0.04, 3), dict(max_len=8, shard_index=1, shard_count=3,
                                                                          min_shard_paths=16)),
    ("gnp600 count (wide class)", I.gnp(600, 0.01, 5), dict(max_len=8)),
    ("gnp600 count shard 0/2 (wide filter)", I.gnp(600, 0.01, 5), dict(max_len=7, shard_index=0, shard_count=2,
                                                                        min_shard_paths=16)),
    ("p5x6 count (small-frontier cooperative kernel)", I.grid(5, 6), {}),
    ("p6x7 count K=12 (blocked LEAF variant)", I.grid(6, 7), dict(max_len=12)),
    ("gnp600 count K=7 (wide bitset + k_leaf_wide)", I.gnp(600, 0.01, 5), dict(max_len=7, record_format=1)),
    ("gnp700 count K=8 (list class + list leaf)", I.gnp(700, 0.008, 11), dict(max_len=8, record_format=2)),
    ("grid24x24 count K=13 (list class, 3 id words)", I.grid(24, 24), dict(max_len=13, record_format=2)),
    ("gnp700 count K=8 shard 1/2 (list filter)", I.gnp(700, 0.008, 11), dict(max_len=8, record_format=2, shard_index=1,
                                                                            shard_count=2, min_shard_paths=16)),
    # round 2 kernels (environment switches force them on small graphs)
    ("grid7x10 count (k_expand_fq, two levels, packed)", I.grid(7, 10), dict(env={"CC_FUSED_MIN": "1", "CC_NO_SMALL": "1"})),
    ("grid7x8 count (k_expand_fused, two levels, unpacked)", I.grid(7, 8), dict(env={"CC_FUSED_MIN": "1", "CC_NO_SMALL": "1"})),
    ("grid7x10 count K=14 (k_expand_fused, single level + leaf)", I.grid(7, 10),
     dict(max_len=14, env={"CC_FUSED_MIN": "1", "CC_NO_SMALL": "1", "CC_FQ": "0"})),
    ("grid7x10 count K=15 shard 1/2 (fused output with empty slots -> filter)", I.grid(7, 10),
     dict(max_len=15, shard_index=1, shard_count=2, min_shard_paths=1 << 12, env={"CC_FUSED_MIN": "1"})),
    ("k60x70 count (Stage 1 chained with the first expansion)", I.complete_bipartite(60, 70), {}),
    ("p8x8 count (small-frontier kernel over page regions)", I.grid(8, 8), {}),
]
bad = 0
for name, g, kw in cases:
    kw = dict(kw)
    env = kw.pop("env", {})
    os.environ.update(env)
    try:
        got = binding.enumerate_cycles(*g, workspace=ws, **kw)
    finally:
        for k in env:
            del os.environ[k]
    okw = {k: v for k, v in kw.items() if k in ("max_len", "collect")}
    if "shard_count" in kw:
        print(name, "ran; cycles on this shard:", int(got["counts"].sum()))
        continue
    want = oracle.enumerate_cycles(*g, **okw)
    same = got["counts"].tolist() == want["counts"].tolist() and got["set_hash"] == want["set_hash"]
    print(name, "OK" if same else "MISMATCH", int(got["counts"].sum()))
    bad += not same
sys.exit(1 if bad else 0)
