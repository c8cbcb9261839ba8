#!/bin/bash
# Round-2 evidence, part B: ncu launch list of the P10x10 bench step and --set full captures of the
# dominant kernels, summarised ON THE BOX (the .ncu-rep files are deleted: gpurun returns <= 64 MiB)
O=gpurun_out/finalB
mkdir -p $O
python -c "from paper_1410_4876_b200 import build; build.build()" > $O/build.log 2>&1
summ() {  # $1 = report basename
  python tools/ncu_summary.py full $O/$1.ncu-rep > $O/$1.summary.txt 2>&1
  ncu -i $O/$1.ncu-rep --page source --csv --print-source=cuda,sass > $O/$1.src.csv 2>/dev/null
  python tools/ncu_lines.py $O/$1.src.csv 60 > $O/$1.lines.txt 2>&1
  ncu -i $O/$1.ncu-rep --page raw --csv > $O/$1.raw.csv 2>/dev/null
}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_p10x10.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
CC_TRACE=$O/trace_fq.csv timeout 900 ncu --nvtx --nvtx-include "expand L44 f2/" --nvtx-include "expand L45 f2/" -c 1 \
    --set full --clock-control none --import-source on -o $O/prof_fq python tools/run_once.py p10x10 > $O/ncu_fq.log 2>&1
summ prof_fq
python tools/traffic_json.py p10x10 $O/prof_fq.ncu-rep $O/trace_fq.csv --level 44 45 --kernel 'k_expand_fq<2>' \
    --record-bytes 24 --r-alg 16 --out $O/ncu_traffic.json > $O/traffic.log 2>&1
timeout 600 ncu -k regex:k_expand_blocked -c 1 --set full --clock-control none --import-source on \
    -o $O/prof_k150 python tools/run_once.py k150 > $O/ncu_k150.log 2>&1
summ prof_k150
timeout 600 ncu -k regex:k_small_levels -c 1 --set full --clock-control none --import-source on \
    -o $O/prof_p8x8_small python tools/run_once.py p8x8 > $O/ncu_p8x8.log 2>&1
summ prof_p8x8_small
CC_TRACE=$O/trace_gnp.csv timeout 900 ncu --nvtx --nvtx-include "expand L8 f0/" -c 1 --set full --clock-control none --import-source on \
    -o $O/prof_list_leaf python tools/run_once.py gnp2000 --max-len 10 > $O/ncu_list.log 2>&1
summ prof_list_leaf
rm -f $O/*.ncu-rep
ls -la $O
du -sh $O
