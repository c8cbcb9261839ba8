#!/bin/bash
# A/B of library variants on G(2000) K=10 (device time, expansion time), e2e probe
mkdir -p gpurun_out
for lib in paper_1410_4876_b200/libchordless.so variants/*.so; do
  echo "== $lib"
  CC_LIBCHORDLESS=$lib timeout 300 python tools/run_once.py gnp2000 --max-len 10 --profile --repeat 4 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l); print(round(d['t_dev_ms'],2), round(d['t_expand_ms'],2), d['hash'], d['cycles'])
    except Exception: print(l.strip()[:200])
"
done
timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1; cat gpurun_out/e2e_probe.log | tail -4
