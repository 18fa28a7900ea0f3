#!/bin/bash
# developer A/B of two prebuilt libraries (ab/libA.so, ab/libB.so) on one box: headline bench
# value (and the output-pass phase), alternating; then the T = 8 slice step
export PYTHONPATH=.
for rep in 1 2 3; do
  for v in A B; do
    val=$(LMOE_LIB=ab/lib$v.so python bench.py --no-extra --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); ph=d['phase_ms_per_step']; print('%.1f M tok/s  %.4f ms  state %.4f  out %.4f' % (d['value']/1e6, d['ms_per_step'], ph.get('state_pass', 0), ph.get('output_pass', 0)))")
    echo "$v bench: $val"
  done
done
if [ "$1" = "slice" ]; then
for rep in 1 2; do
  for v in A B; do
    echo "$v slice 32768: $(LMOE_LIB=ab/lib$v.so python tools/sp_overhead_probe.py 32768 2>/dev/null | tail -1)"
  done
done
fi
