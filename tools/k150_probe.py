"""Per-call overhead probe for small workloads (K_{150,150}): device time between torch events
around cc_enumerate (as bench.py times it), the library's own t_dev_ms, and host wall time."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1410_4876_b200 import binding, inputs  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "k150"
g = inputs.named(w)
ws = torch.empty(8 << 30, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
gr = binding.cc_graph_from_csr(*g)
for prof in (False, True):
    opts = binding.make_options(stream=st.cuda_stream, workspace=ws, profile=prof)
    for _ in range(5):
        binding.cc_enumerate(gr, opts)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    tdev, walls = [], []
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for a, b in ev:
        flush.zero_()
        a.record(st)
        t0 = time.perf_counter()
        r = binding.cc_enumerate(gr, opts)
        walls.append((time.perf_counter() - t0) * 1e3)
        b.record(st)
        tdev.append(binding.cc_result_stats(r)["t_dev_ms"])
    torch.cuda.synchronize()
    evms = sorted(a.elapsed_time(b) for a, b in ev)
    print(f"{w} profile={prof}: event ms median {evms[10]:.4f} min {evms[0]:.4f}; lib t_dev median "
          f"{sorted(tdev)[10]:.4f}; host wall median {sorted(walls)[10]:.4f} ms")
