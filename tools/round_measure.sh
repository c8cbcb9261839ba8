#!/bin/bash
# One GPU session of round-end evidence (run under gpurun from the repo root):
#   tests, smoke, bench lines for the main workloads, ncu launch list + one --set full capture
#   of the dominant kernel (with the CC_TRACE of the same deterministic run), list-class capture.
# Everything lands in gpurun_out/; tools/ncu_summary.py and tools/traffic_json.py turn it into
# profiles/ files on the CPU box.
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_p10x10.json 2> gpurun_out/bench_p10x10.err
for w in k150 p8x8 gnp2000k10 gnp2000k11; do
  python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_p10.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
CC_TRACE=gpurun_out/trace_p10.csv python tools/run_once.py p10x10 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_expand_blocked -s 45 -c 1 \
    -o gpurun_out/prof_eb_final python tools/run_once.py p10x10 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_expand_list -c 6 \
    -o gpurun_out/prof_list_final python tools/run_once.py gnp2000 --max-len 10 > /dev/null 2>&1
ls -la gpurun_out
