#!/bin/bash
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
export PYTHONPATH=.
for rep in 1 2; do
  for pf in 0 1 2; do echo "PF=$pf $(LMOE_VB_PF=$pf timeout 120 python tools/bwd_vec_time.py x 262144 gla 2>&1 | tail -1)"; done
done
timeout 900 python -m pytest tests/test_lsm_bwd_gpu.py -q -x 2>&1 | tail -3
