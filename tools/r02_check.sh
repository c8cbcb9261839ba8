#!/bin/bash
# Round-2 check: full GPU suite, smoke, default bench line, and the N > 1 path on one GPU.
mkdir -p gpurun_out
python -c "from paper_1410_4876_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_p10x10.json 2> gpurun_out/bench_p10x10.err
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --workspace-gb 60 > gpurun_out/bench_p10x10_g2.json 2> gpurun_out/bench_p10x10_g2.err
tail -c 600 gpurun_out/bench_p10x10_g2.err
ls -la gpurun_out
