#!/bin/bash
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
timeout 600 python -m pytest tests/test_lsm_bwd_gpu.py -q -x -k "vector" 2>&1 | tail -25
PYTHONPATH=. timeout 300 python tools/bwd_vec_time.py 2>&1 | tail -5
PYTHONPATH=. timeout 300 python tools/bwd_vec_time.py t 262144 hgrn2 2>&1 | tail -5
