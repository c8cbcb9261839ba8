#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_1410_4876_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or full_size or shard" > gpurun_out/pytest_fused.log 2>&1
rc=$?; tail -3 gpurun_out/pytest_fused.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_p10x10.json 2> gpurun_out/bench_p10x10.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_p10x10.json"))
print(d["ms_per_step"], d["set_hash"], d["roofline"]["frac"], d["roofline"].get("frac_moved"), d["gpu_launches"])
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_expand_fused -s 30 -c 1 \
    -o gpurun_out/prof_fused_b python tools/run_once.py p10x10 > gpurun_out/ncu_fused.log 2>&1
