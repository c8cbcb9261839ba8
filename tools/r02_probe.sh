#!/bin/bash
# Round-2 first probe: GPU tests, one bench line, ncu source-level capture of the dominant kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_p10x10.json 2> gpurun_out/bench_p10x10.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_expand_blocked -s 40 -c 1 \
    -o gpurun_out/prof_eb_r02a python tools/run_once.py p10x10 > gpurun_out/ncu_eb.log 2>&1
ls -la gpurun_out
