#!/bin/bash
# round-2 A/B: in-tree library (new) against variants/*.so on P10x10, after the fused-kernel tests
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout 120 -k "fused or full_size or small_frontier or chunked" > gpurun_out/pytest_ab7.log 2>&1
rc=$?; tail -2 gpurun_out/pytest_ab7.log; if [ $rc -ne 0 ]; then exit 1; fi
bash tools/r02_ab5.sh ${1:-p10x10}
