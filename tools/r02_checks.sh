#!/bin/bash
# Debug build with device-side bounds checks in k_expand_fq (-DCC_CHECKS): the substitute for
# compute-sanitizer, which the GPU pool has disabled.  The self-test build must fail (the check
# plumbing works); the checked build must pass the fused / chunked / sharded / full-size tests.
O=gpurun_out/checks
mkdir -p $O
CC_LIBCHORDLESS=variants/checks_selftest.so timeout 300 python -c "
import torch
from paper_1410_4876_b200 import binding, inputs as I
ws = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
import os; os.environ['CC_FUSED_MIN'] = '1'; os.environ['CC_NO_SMALL'] = '1'
try:
    binding.enumerate_cycles(*I.grid(7, 10), workspace=ws)
    print('SELFTEST: check did NOT fire')
except Exception as e:
    print('SELFTEST: check fired as expected:', e)
" > $O/selftest.log 2>&1; cat $O/selftest.log | tail -1
CC_LIBCHORDLESS=variants/checks.so timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_multigpu_gpu.py -q \
   -k "fused or chunked or shard or full_size or small_frontier or packed or p8x8 or table1 or p10x10" > $O/pytest_checks.log 2>&1
tail -2 $O/pytest_checks.log
CC_LIBCHORDLESS=variants/checks.so timeout 600 python tools/run_once.py p10x10 > $O/p10x10_checks.log 2>&1; tail -1 $O/p10x10_checks.log
