#!/bin/bash
# k_expand_blocked A/B: its parity tests, then K_{150,150} device time per variant
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "k150 or word_boundaries or dense or table1 or max_len or shards or chained or k50" > gpurun_out/pytest_abk.log 2>&1
rc=$?; tail -2 gpurun_out/pytest_abk.log; if [ $rc -ne 0 ]; then exit 1; fi
bash tools/r02_abw.sh k150 0 5
