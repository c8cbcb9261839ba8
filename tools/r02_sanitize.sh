#!/bin/bash
mkdir -p gpurun_out/san
python -c "from paper_1410_4876_b200 import build; build.build()" > gpurun_out/san/build.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/san/$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/san/$tool.log
  tail -3 gpurun_out/san/$tool.log
done
