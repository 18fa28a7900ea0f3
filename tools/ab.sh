#!/bin/bash
# developer A/B of two prebuilt libraries (ab/libA.so, ab/libB.so) on one box: headline bench
# value and the T = 8 slice step, alternating
export PYTHONPATH=.
for rep in 1 2; do
  for v in A B; do
    val=$(LMOE_LIB=ab/lib$v.so python bench.py --no-extra --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.1f M tok/s  %.4f ms' % (d['value']/1e6, d['ms_per_step']))")
    echo "$v bench: $val"
  done
done
for rep in 1 2; do
  for v in A B; do
    echo "$v slice 32768: $(LMOE_LIB=ab/lib$v.so python tools/sp_overhead_probe.py 32768 2>/dev/null | tail -1)"
  done
done
