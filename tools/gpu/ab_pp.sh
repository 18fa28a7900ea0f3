#!/bin/bash
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
export PYTHONPATH=.
timeout 600 python -m pytest tests/test_attn_gpu.py tests/test_nccl_gpu.py tests/test_model_gpu.py -q -x 2>&1 | tail -3
for rep in 1 2; do
  for v in 0 1; do echo "PP=$v $(LMOE_ATTN_PP=$v timeout 120 python tools/bench_attn.py 0 3 7 2>&1 | tr '\n' ' ')"; done
done
