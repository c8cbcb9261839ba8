#!/bin/bash
# list-class A/B: parity tests of the list kernels, then G(2000, 0.005) K = 10 and K = 11
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "gnp or list or wide or full_size" > gpurun_out/pytest_ablist.log 2>&1
rc=$?; tail -2 gpurun_out/pytest_ablist.log; if [ $rc -ne 0 ]; then exit 1; fi
bash tools/r02_abw.sh gnp2000 10 3
bash tools/r02_abw.sh gnp2000 11 2
