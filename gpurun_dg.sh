#!/bin/bash
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
export PYTHONPATH=.
timeout 600 python -m pytest tests/test_lsm_bwd_gpu.py -q 2>&1 | tail -3
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mamba2 bwd', d['backward']['ms_per_step'], 'gla', d['gla']['forward']['ms_per_step'], d['gla']['backward']['ms_per_step'])"
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:lsm_mamba_dgate python tools/bwd_once.py 2>&1 | grep -E "lsm_mamba_dgate|gpu__time" | head -4
