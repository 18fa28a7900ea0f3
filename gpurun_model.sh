#!/bin/bash
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
timeout 300 python -m pytest tests/test_model_gpu.py -q -x 2>&1 | grep -E "Error|error|assert|passed|failed" | head -30
