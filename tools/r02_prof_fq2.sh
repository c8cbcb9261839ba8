#!/bin/bash
# per-launch trace of P10x10 and one ncu --set full capture of the level-45 k_expand_fq launch
O=gpurun_out/pfq
mkdir -p $O
python -c "from paper_1410_4876_b200 import build; build.build()" > $O/build.log 2>&1
CC_TRACE=$O/trace.csv timeout 300 python tools/run_once.py p10x10 --profile > $O/run.log 2>&1
CC_TRACE=$O/trace_ncu.csv timeout 900 ncu --nvtx --nvtx-include "expand L45 f2/" -c 1 \
    --set full --clock-control none --import-source on -o $O/prof_fq python tools/run_once.py p10x10 > $O/ncu_fq.log 2>&1
python tools/ncu_summary.py full $O/prof_fq.ncu-rep > $O/prof_fq.summary.txt 2>&1
ncu -i $O/prof_fq.ncu-rep --page source --csv --print-source=cuda,sass > $O/prof_fq.src.csv 2>/dev/null
python tools/ncu_lines.py $O/prof_fq.src.csv 60 > $O/prof_fq.lines.txt 2>&1
python tools/traffic_json.py p10x10 $O/prof_fq.ncu-rep $O/trace_ncu.csv --level 45 --kernel 'k_expand_fq<2>' \
    --record-bytes 24 --r-alg 16 --out $O/ncu_traffic.json > $O/traffic.log 2>&1
rm -f $O/prof_fq.src.csv
ls -la $O
