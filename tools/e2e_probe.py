import time, torch, sys
sys.path.insert(0, '/root/repo')
from paper_1410_4876_b200 import binding, inputs
g = inputs.named('gnp2000')
free, _ = torch.cuda.mem_get_info()
ws = torch.empty(int(free * 0.85) - (1 << 30), dtype=torch.uint8, device='cuda')
st = torch.cuda.current_stream().cuda_stream
for i in range(4):
    t0 = time.perf_counter(); gr = binding.cc_graph_from_csr(*g); t1 = time.perf_counter()
    r = binding.cc_enumerate(gr, workspace=ws, max_len=10, stream=st); t2 = time.perf_counter()
    c, h = binding.cc_count_by_length(r); t3 = time.perf_counter()
    s = binding.cc_result_stats(r)
    del r; del gr; torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"graph {1e3*(t1-t0):.2f} ms  enumerate {1e3*(t2-t1):.2f} ms (dev {s['t_dev_ms']:.2f}, wall {s['t_wall_ms']:.2f})  counts {1e3*(t3-t2):.2f}  free {1e3*(t4-t3):.2f}")
