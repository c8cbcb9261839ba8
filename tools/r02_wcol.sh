#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_1410_4876_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "wide_collect or collect_at_scale or too_large or gnp2000_config3 or list_class or wide_class" > gpurun_out/pytest_wcol.log 2>&1
rc=$?; tail -3 gpurun_out/pytest_wcol.log
if [ $rc -ne 0 ]; then grep -E "Error|assert" gpurun_out/pytest_wcol.log | head -20; fi
timeout 300 python bench.py --workload gnp2000k10 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_gnp10.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/bench_gnp10.json')); print('gnp2000k10', d['ms_per_step'], d['set_hash'])"
