#!/bin/bash
export PYTHONPATH=$PWD:$PYTHONPATH
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
timeout 300 python tools/fused_chain_check.py 40000 16 30 | grep -E "[1-9] bad|rep 29"
timeout 200 python tools/fused_race.py 262144 16 6 mamba2
timeout 200 python tools/fused_race.py 262144 16 2 bla_plain
timeout 900 python -m pytest tests/test_fused_gpu.py -q -x 2>&1 | tail -3
