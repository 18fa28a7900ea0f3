#!/bin/bash
# fused-forward timeline + its tests
export PYTHONPATH=$PWD:$PYTHONPATH
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
timeout 300 python tools/dbg_fused.py 40000 16 1
timeout 300 python tools/dbg_fused.py 40000 16 0
timeout 120 python tools/trace_fused.py 2>&1 | tail -70
LMOE_FUSED_SEGC=4 timeout 120 python tools/trace_fused.py 2>&1 | grep -E "plan|call|medians"
LMOE_FUSED_SEGC=16 timeout 120 python tools/trace_fused.py 2>&1 | grep -E "plan|call|medians"
LMOE_FUSED_HINT=0 timeout 120 python tools/trace_fused.py 2>&1 | grep -E "plan|call|medians"
