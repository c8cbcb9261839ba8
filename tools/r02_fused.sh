#!/bin/bash
# fused-kernel check: targeted parity tests first (stop on failure), then bench lines
mkdir -p gpurun_out
python -c "from paper_1410_4876_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused" > gpurun_out/pytest_fused.log 2>&1
rc=$?; tail -3 gpurun_out/pytest_fused.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_p10x10.json 2> gpurun_out/bench_p10x10.err
timeout 300 python bench.py --workload p8x8 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_p8x8.json 2> gpurun_out/bench_p8x8.err
CC_NO_FUSED=1 timeout 300 python bench.py --workload p8x8 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_p8x8_nofused.json 2>&1
python - <<'PY'
import json
for f in ["bench_p10x10", "bench_p8x8", "bench_p8x8_nofused"]:
    try:
        d = json.load(open(f"gpurun_out/{f}.json"))
        print(f, d["ms_per_step"], d["set_hash"], d["roofline"]["frac"], d["roofline"].get("frac_moved"), d["gpu_launches"])
    except Exception as e:
        print(f, "ERR", e)
PY
