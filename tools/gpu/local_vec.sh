#!/bin/bash
# TokenVector local-state forward: parity, then GLA cfg3 forward A/B (LMOE_LOCAL_VEC=0/1)
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
export PYTHONPATH=.
timeout 1200 python -m pytest tests/test_local_gpu.py tests/test_lsm_gpu.py tests/test_sp_gpu.py tests/test_model_gpu.py -q -x 2>&1 | grep -v "^  " | tail -12
for rep in 1 2; do
  for f in 0 1; do
    echo "LOCAL_VEC=$f $(LMOE_LOCAL_VEC=$f timeout 300 python -c "
import json, torch, bench
r = bench.gla_bench(torch.device('cuda:0'), steps=10, warmup=3)
print('fwd %.4f ms (%.3f of HBM)  bwd %.4f ms' % (r['forward']['ms_per_step'], r['forward']['roofline']['frac'], r['backward']['ms_per_step']))
")"
  done
done
