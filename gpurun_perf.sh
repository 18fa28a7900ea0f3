#!/bin/bash
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | grep -E "Error|assert|passed|failed" | head -20
timeout 300 python bench.py --no-cpu-baseline --no-extra --steps 10 --warmup 3 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e6, 'Mtok/s', d['roofline']['frac'], d['phase_ms_per_step'])"
