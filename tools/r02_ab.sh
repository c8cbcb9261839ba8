#!/bin/bash
# A/B of expansion variants on P10x10: per-level times from the library trace
mkdir -p gpurun_out
python -c "from paper_1410_4876_b200 import build; build.build()" > gpurun_out/build.log 2>&1
for v in "fmin24:CC_FUSED_MIN=16777216" "fmin20:CC_FUSED_MIN=1048576" "nofused:CC_NO_FUSED=1"; do
  name=${v%%:*}; envs=${v#*:}
  rm -f gpurun_out/trace_$name.csv
  env $envs CC_TRACE=gpurun_out/trace_$name.csv timeout 300 python tools/run_once.py p10x10 --profile --repeat 2 > gpurun_out/run_$name.log 2>&1
  echo "== $name"; tail -1 gpurun_out/run_$name.log
done
