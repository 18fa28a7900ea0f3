#!/bin/bash
# dgate A/B: B = previous candidate, C = candidate
export PYTHONPATH=.
timeout 900 python -m pytest tests/test_lsm_bwd_gpu.py -q -x 2>&1 | grep -v "^  " | tail -3
sed -n '/^cat > \/tmp\/bwdt.py/,/^PY$/p' tools/gpu/ab_bwd.sh | sed '1d;$d' > /tmp/bwdt.py
for rep in 1 2; do
  echo "B  $(LMOE_LIB=ab/libB.so timeout 120 python /tmp/bwdt.py 2>&1 | tail -1)"
  echo "C  $(LMOE_LIB=ab/libC.so timeout 120 python /tmp/bwdt.py 2>&1 | tail -1)"
done
NCU=/usr/local/cuda/bin/ncu
LMOE_LIB=ab/libC.so timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/dgate_C.csv python tools/bwd_once.py > /dev/null 2>&1
python tools/launch_table.py gpurun_out/dgate_C.csv 2>/dev/null | grep -i "dgate"
LMOE_LIB=ab/libC.so timeout 900 $NCU --set full --clock-control none --import-source on -k regex:lsm_mamba_dgate -s 1 -c 1 \
   -o gpurun_out/r2_prof_dgate python tools/bwd_once.py > /dev/null 2>&1
