#!/bin/bash
# dgate A/B: A = previous library, B = candidate, B0 = candidate without the L2 prefetch
export PYTHONPATH=.
timeout 900 python -m pytest tests/test_lsm_bwd_gpu.py -q -x 2>&1 | grep -v "^  " | tail -3
sed -n '/^cat > \/tmp\/bwdt.py/,/^PY$/p' tools/gpu/ab_bwd.sh | sed '1d;$d' > /tmp/bwdt.py
for rep in 1 2; do
  echo "A  $(LMOE_LIB=ab/libA.so timeout 120 python /tmp/bwdt.py 2>&1 | tail -1)"
  echo "B  $(LMOE_LIB=ab/libB.so timeout 120 python /tmp/bwdt.py 2>&1 | tail -1)"
  echo "B0 $(LMOE_DG_PF=0 LMOE_LIB=ab/libB.so timeout 120 python /tmp/bwdt.py 2>&1 | tail -1)"
done
NCU=/usr/local/cuda/bin/ncu
for pf in 1 0; do
LMOE_DG_PF=$pf LMOE_LIB=ab/libB.so timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/dgate_B$pf.csv python tools/bwd_once.py > /dev/null 2>&1
echo "pf=$pf"; python tools/launch_table.py gpurun_out/dgate_B$pf.csv 2>/dev/null | grep -i "dgate"
done
