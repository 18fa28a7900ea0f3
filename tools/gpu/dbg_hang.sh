#!/bin/bash
export PYTHONPATH=.
for a in "retnet 2305" "retnet 1153" "retnet 1152" "bla 2305"; do
  echo "=== $a"; CUDA_LAUNCH_BLOCKING=1 timeout 60 python tools/dbg_hang.py $a 2>&1 | tail -4
done
echo "=== LMOE_LOCAL=0 retnet 2305"; LMOE_LOCAL=0 CUDA_LAUNCH_BLOCKING=1 timeout 60 python tools/dbg_hang.py retnet 2305 2>&1 | tail -3
timeout 300 python -m pytest tests/test_tensor_bridge_gpu.py -q -p no:cacheprovider 2>&1 | grep -i "fail\|error" | head -10
