#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_1410_4876_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "chained or k150 or fused or small_frontier" > gpurun_out/pytest_chain.log 2>&1
rc=$?; tail -2 gpurun_out/pytest_chain.log
if [ $rc -ne 0 ]; then grep -E "Error|assert" gpurun_out/pytest_chain.log | head; exit 1; fi
timeout 300 python bench.py --workload k150 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_k150.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/bench_k150.json')); print('k150', d['ms_per_step'], d['ms_per_step_median'], d['set_hash'], d['gpu_launches']/d['steps'], d['e2e']['ms_per_step'])"
for lib in paper_1410_4876_b200/libchordless.so variants/*.so; do
  echo "== $lib"
  CC_LIBCHORDLESS=$lib timeout 300 python tools/run_once.py p10x10 --repeat 3 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l); print(round(d['t_dev_ms'],1), d['hash'], d['launches'])
    except Exception: print(l.strip()[:200])
"
done
