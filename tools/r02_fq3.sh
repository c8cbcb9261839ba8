#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_1410_4876_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or full_size or small_frontier or chunked" > gpurun_out/pytest_fq.log 2>&1
rc=$?; tail -2 gpurun_out/pytest_fq.log
if [ $rc -ne 0 ]; then grep -E "Error|assert" gpurun_out/pytest_fq.log | head; exit 1; fi
timeout 300 python tools/run_once.py p10x10 --repeat 3 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l); print(round(d['t_dev_ms'],1), d['hash'], d['launches'])
    except Exception: print(l.strip()[:200])
"
