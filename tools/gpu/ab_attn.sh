#!/bin/bash
export PYTHONPATH=.
for rep in 1 2; do
  for v in A B; do echo "$v $(LMOE_LIB=ab/lib$v.so timeout 120 python tools/bench_attn.py 0 7 2>&1 | tr '\n' ' ')"; done
done
timeout 600 python -m pytest tests/test_attn_gpu.py tests/test_nccl_gpu.py -q -x 2>&1 | tail -2
