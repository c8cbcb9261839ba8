#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_1410_4876_b200 import build; build.build()" > gpurun_out/build.log 2>&1
CC_TRACE=gpurun_out/trace_fused.csv timeout 300 python tools/run_once.py p10x10 --profile > gpurun_out/run_once.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_expand_fused -s 30 -c 1 \
    -o gpurun_out/prof_fused_a python tools/run_once.py p10x10 > gpurun_out/ncu_fused.log 2>&1
tail -3 gpurun_out/ncu_fused.log
timeout 600 python -m pytest tests/test_multigpu_gpu.py -q -x > gpurun_out/pytest_mgpu.log 2>&1; tail -2 gpurun_out/pytest_mgpu.log
