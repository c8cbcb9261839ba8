#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_1410_4876_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or full_size" > gpurun_out/pytest_ab6.log 2>&1
rc=$?; tail -2 gpurun_out/pytest_ab6.log; if [ $rc -ne 0 ]; then exit 1; fi
bash tools/r02_ab5.sh p10x10
