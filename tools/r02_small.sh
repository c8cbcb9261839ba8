#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_1410_4876_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small_frontier or full_size or chunked or table1 or max_len or fused" > gpurun_out/pytest_small.log 2>&1
rc=$?; tail -3 gpurun_out/pytest_small.log
if [ $rc -ne 0 ]; then exit 1; fi
for w in p8x8 k150 p4x4; do
timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
python - <<'PY'
import json
for w in ["p8x8", "k150", "p4x4"]:
    d = json.load(open(f"gpurun_out/bench_{w}.json"))
    print(w, d["ms_per_step"], d["ms_per_step_median"], d["set_hash"], d["gpu_launches"] / d["steps"], d["e2e"]["ms_per_step"], d["roofline"]["frac"])
PY
