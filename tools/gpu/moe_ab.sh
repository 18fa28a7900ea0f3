#!/bin/bash
# MoE permute A/B: A = dispatch-order gather, B = token-order scatter (in-tree library = B)
export PYTHONPATH=.
timeout 1200 python -m pytest tests/test_moe_gpu.py tests/test_model_gpu.py tests/test_determinism_gpu.py "tests/test_fullshape_gpu.py::test_cfg4_moe_full_shape" -q -x 2>&1 | grep -v "^  " | tail -3
for rep in 1 2 3; do for v in A B; do
  echo "$v $(LMOE_LIB=ab/lib$v.so timeout 120 python tools/bench_moe.py 2>&1 | tail -1)"
done; done
NCU=/usr/local/cuda/bin/ncu
for v in A B; do
LMOE_LIB=ab/lib$v.so STEPS=1 timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/moe_$v.csv python tools/bench_moe.py > /dev/null 2>&1
echo "== $v"; python tools/launch_table.py gpurun_out/moe_$v.csv 2>/dev/null | grep "lmoe"
done
