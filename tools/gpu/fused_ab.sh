#!/bin/bash
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
export PYTHONPATH=.
timeout 900 python -m pytest tests/test_fused_gpu.py -q -x 2>&1 | grep -v "^  " | tail -12
for rep in 1 2; do
  for f in 0 1; do
    echo "FUSED=$f $(LMOE_FUSED=$f timeout 300 python bench.py --no-cpu-baseline --no-extra --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.1f M tok/s %.4f ms' % (d['value']/1e6, d['ms_per_step']), d['roofline']['plan'])")"
  done
done
for c in 4 6 8 12; do
  echo "SEGC=$c $(LMOE_FUSED=1 LMOE_FUSED_SEGC=$c timeout 300 python bench.py --no-cpu-baseline --no-extra --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.1f M tok/s %.4f ms' % (d['value']/1e6, d['ms_per_step']), d['roofline']['plan'])")"
done
LMOE_FUSED=1 timeout 120 python tools/trace_fused.py 2>&1 | tail -25
