#!/bin/bash
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
export PYTHONPATH=.
timeout 300 python tools/bwd_vec_time.py 2>&1 | tail -2
timeout 300 python tools/trace_vec.py gla 2>&1 | tail -6
timeout 300 python tools/trace_vbc.py 65536 2>&1 | tail -3
