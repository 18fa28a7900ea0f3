#!/bin/bash
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | grep -v "^  " | tail -8
timeout 600 python bench.py 2>gpurun_out/bench_err.log | tee gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 2>gpurun_out/bench_ref_err.log | tee gpurun_out/bench_ref.json
tail -3 gpurun_out/bench_err.log gpurun_out/bench_ref_err.log
