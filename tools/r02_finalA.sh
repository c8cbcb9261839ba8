#!/bin/bash
# Round-2 evidence, part A: GPU suite, smoke, bench lines for every workload, N=2 on one GPU
O=gpurun_out/finalA
mkdir -p $O
python -c "from paper_1410_4876_b200 import build; build.build()" > $O/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -3 $O/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_p10x10.json 2> $O/bench_p10x10.err
for w in k150 p8x8 p4x4 grid8x10 gnp2000 gnp2000k10 gnp2000k11; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --workspace-gb 60 --no-cpu-baseline > $O/bench_p10x10_g2.json 2> $O/bench_p10x10_g2.err
timeout 600 python tools/run_once.py k150 --collect --repeat 2 > $O/collect_k150.log 2>&1
ls -la $O
timeout 900 python tools/shard_balance.py p10x10 --shards 2 4 8 > $O/shard_balance.jsonl 2> $O/shard_balance.err
timeout 600 python tools/shard_balance.py gnp2000 --max-len 10 --shards 2 4 8 >> $O/shard_balance.jsonl 2>> $O/shard_balance.err
timeout 600 python tools/shard_balance.py k150 --shards 2 4 8 >> $O/shard_balance.jsonl 2>> $O/shard_balance.err
tail -c 1500 $O/shard_balance.jsonl
