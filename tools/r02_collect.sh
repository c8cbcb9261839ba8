#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_1410_4876_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "collect" > gpurun_out/pytest_collect.log 2>&1
tail -3 gpurun_out/pytest_collect.log
timeout 300 python tools/run_once.py k150 --collect --repeat 2 > gpurun_out/collect_k150.log 2>&1; tail -2 gpurun_out/collect_k150.log
CC_TRACE=gpurun_out/trace_k150.csv timeout 300 python tools/run_once.py k150 --profile --repeat 3 > gpurun_out/k150_once.log 2>&1; tail -1 gpurun_out/k150_once.log
tail -4 gpurun_out/trace_k150.csv
