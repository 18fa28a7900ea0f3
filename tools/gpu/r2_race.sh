#!/bin/bash
export PYTHONPATH=$PWD:$PYTHONPATH
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | grep -v "^  " | tail -6
timeout 300 python bench.py --no-cpu-baseline --no-extra 2>gpurun_out/bench_err.log | tee gpurun_out/bench.json
