#!/bin/bash
# GPU suite + smoke + default bench line (P10x10)
O=gpurun_out/suite
mkdir -p $O
python -c "from paper_1410_4876_b200 import build; build.build()" > $O/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -3 $O/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_p10x10.json 2> $O/bench_p10x10.err
cat $O/bench_p10x10.json | head -c 600
