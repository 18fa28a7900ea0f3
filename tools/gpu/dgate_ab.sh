#!/bin/bash
# persistent dgate: backward tests (library in-tree = B), A/B timing, dgate launch times
export PYTHONPATH=.
timeout 900 python -m pytest tests/test_lsm_bwd_gpu.py -q -x 2>&1 | grep -v "^  " | tail -5
bash tools/gpu/ab_bwd.sh
NCU=/usr/local/cuda/bin/ncu
for v in A B; do
LMOE_LIB=ab/lib$v.so timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/dgate_$v.csv python tools/bwd_once.py > /dev/null 2>&1
python tools/launch_table.py gpurun_out/dgate_$v.csv 2>/dev/null | grep -i "dgate\|output_pass\|state_pass"
done
