#!/bin/bash
# ncu --set full of exactly the first expansion of level 44 of P10x10 (CC_PROFILE_LEVEL), fused
# kernel and (CC_NO_FUSED) the single-level kernel, with the library trace of the same run
mkdir -p gpurun_out
python -c "from paper_1410_4876_b200 import build; build.build()" > gpurun_out/build.log 2>&1
tag=${1:-x}
CC_TRACE=gpurun_out/trace44_$tag.csv timeout 900 ncu --nvtx --nvtx-include "expand L44 f2/" --nvtx-include "expand L45 f2/" -c 1 --set full --clock-control none --import-source on \
    -o gpurun_out/prof44_$tag python tools/run_once.py p10x10 > gpurun_out/ncu44_$tag.log 2>&1
tail -2 gpurun_out/ncu44_$tag.log
if [ "$2" == "old" ]; then
CC_NO_FUSED=1 CC_TRACE=gpurun_out/trace44_old.csv timeout 900 ncu --nvtx --nvtx-include "expand L44 f0/" -c 1 --set full --clock-control none --import-source on \
    -o gpurun_out/prof44_old python tools/run_once.py p10x10 > gpurun_out/ncu44_old.log 2>&1
tail -2 gpurun_out/ncu44_old.log
fi
