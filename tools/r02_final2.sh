#!/bin/bash
# last refresh after the branch-free test: GPU suite, smoke, bounds-checked build, P10x10 and
# Grid 8x10 bench lines, ncu of the level-45 launch
O=gpurun_out/f2
mkdir -p $O
python -c "from paper_1410_4876_b200 import build; build.build()" > $O/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
bash tools/r02_checks.sh > $O/checks.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_p10x10.json 2> $O/bench_p10x10.err
timeout 600 python bench.py --workload grid8x10 --steps 10 --warmup 3 > $O/bench_grid8x10.json 2> $O/bench_grid8x10.err
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --workspace-gb 60 --no-cpu-baseline > $O/bench_p10x10_g2.json 2> $O/bench_p10x10_g2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_p10x10.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
CC_TRACE=$O/trace_fq.csv timeout 900 ncu --nvtx --nvtx-include "expand L45 f2/" -c 1 \
    --set full --clock-control none --import-source on -o $O/prof_fq python tools/run_once.py p10x10 > $O/ncu_fq.log 2>&1
python tools/ncu_summary.py full $O/prof_fq.ncu-rep > $O/prof_fq.summary.txt 2>&1
ncu -i $O/prof_fq.ncu-rep --page source --csv --print-source=cuda,sass > $O/prof_fq.src.csv 2>/dev/null
python tools/ncu_lines.py $O/prof_fq.src.csv 60 > $O/prof_fq.lines.txt 2>&1
rm -f $O/prof_fq.src.csv
python tools/traffic_json.py p10x10 $O/prof_fq.ncu-rep $O/trace_fq.csv --level 45 --kernel 'k_expand_fq<2>' \
    --record-bytes 24 --r-alg 16 --out $O/ncu_traffic.json > $O/traffic.log 2>&1
timeout 900 python tools/shard_balance.py p10x10 --shards 2 4 8 > $O/shard_balance.jsonl 2> $O/shard_balance.err
ls -la $O
