#!/bin/bash
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
export PYTHONPATH=.
timeout 1500 python -m pytest tests/test_local_gpu.py tests/test_determinism_gpu.py tests/test_moe_gpu.py tests/test_lsm_gpu.py tests/test_sp_gpu.py tests/test_nccl_gpu.py tests/test_fullshape_gpu.py -q -x 2>&1 | grep -v "^  " | tail -12
for rep in 1 2; do
  for f in 0 1; do
    echo "LOCAL=$f $(LMOE_LOCAL=$f timeout 300 python bench.py --no-cpu-baseline --no-extra --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.1f M tok/s %.4f ms' % (d['value']/1e6, d['ms_per_step']), {k: round(v,4) for k,v in d['phase_ms_per_step'].items()})")"
  done
done
timeout 300 python tools/sp_scaling_probe.py 2>&1 | tail -8
