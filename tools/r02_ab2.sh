#!/bin/bash
# A/B of library variants on P10x10 (device time per run), plus the G(2000) e2e probe
mkdir -p gpurun_out
for lib in paper_1410_4876_b200/libchordless.so variants/*.so; do
  echo "== $lib"
  CC_LIBCHORDLESS=$lib timeout 300 python tools/run_once.py p10x10 --repeat 3 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l); print(d['t_dev_ms'], d['hash'], d['launches'])
    except Exception: print(l.strip()[:200])
"
done
timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1; cat gpurun_out/e2e_probe.log | tail -4
