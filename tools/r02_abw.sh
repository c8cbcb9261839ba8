#!/bin/bash
# A/B of library variants: $1 = workload, $2 = max_len (0 = none), $3 = repeats
mkdir -p gpurun_out
python -c "from paper_1410_4876_b200 import build; build.build()" > gpurun_out/build.log 2>&1
for lib in paper_1410_4876_b200/libchordless.so variants/*.so; do
  echo "== $lib"
  CC_LIBCHORDLESS=$lib timeout 300 python tools/run_once.py $1 --max-len $2 --repeat $3 --profile 2>&1 | python -c "
import sys, json
r = []
for l in sys.stdin:
    try: d = json.loads(l); r.append((round(d['t_dev_ms'],4), round(d['t_expand_ms'],4), d['hash']))
    except Exception: print(l.strip()[:200])
print(r[-3:])
"
done
