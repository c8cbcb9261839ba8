#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_1410_4876_b200 import build; build.build()" > gpurun_out/build.log 2>&1
for lib in paper_1410_4876_b200/libchordless.so variants/*.so; do
  echo "== $lib"
  CC_LIBCHORDLESS=$lib timeout 300 python tools/run_once.py ${1:-p10x10} --repeat 3 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l); print(round(d['t_dev_ms'],3), d['hash'], d['launches'])
    except Exception: print(l.strip()[:200])
"
done
