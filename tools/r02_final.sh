#!/bin/bash
# Round-2 evidence: GPU suite, smoke, bench lines for every workload, N=2 on one GPU (gloo),
# ncu launch list + --set full captures of the dominant kernels, with the library traces.
O=gpurun_out/final
mkdir -p $O
python -c "from paper_1410_4876_b200 import build; build.build()" > $O/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -3 $O/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_p10x10.json 2> $O/bench_p10x10.err
for w in k150 p8x8 p4x4 grid8x10 gnp2000 gnp2000k10 gnp2000k11; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --workspace-gb 60 --no-cpu-baseline > $O/bench_p10x10_g2.json 2> $O/bench_p10x10_g2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_p10x10.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
CC_TRACE=$O/trace_fq.csv timeout 900 ncu --nvtx --nvtx-include "expand L44 f2/" --nvtx-include "expand L45 f2/" -c 1 \
    --set full --clock-control none --import-source on -o $O/prof_fq python tools/run_once.py p10x10 > $O/ncu_fq.log 2>&1
timeout 600 ncu -k regex:k_expand_blocked -c 1 --set full --clock-control none --import-source on \
    -o $O/prof_k150 python tools/run_once.py k150 > $O/ncu_k150.log 2>&1
timeout 600 ncu -k regex:k_small_levels -c 1 --set full --clock-control none --import-source on \
    -o $O/prof_p8x8_small python tools/run_once.py p8x8 > $O/ncu_p8x8.log 2>&1
CC_TRACE=$O/trace_gnp.csv timeout 900 ncu --nvtx --nvtx-include "expand L8 f0/" -c 1 --set full --clock-control none --import-source on \
    -o $O/prof_list_leaf python tools/run_once.py gnp2000 --max-len 10 > $O/ncu_list.log 2>&1
ls -la $O
