#!/bin/bash
# fused-forward bring-up: its tests (each under a timeout), then the bench headline
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
rm -f gpurun_out/parity_errors.jsonl
timeout 300 python -m pytest tests/test_fused_gpu.py -q -x -k "N1 or N129" 2>&1 | tail -5
timeout 600 python -m pytest tests/test_fused_gpu.py -q -x 2>&1 | tail -5
timeout 300 python bench.py --no-cpu-baseline --no-extra 2>gpurun_out/bench_err.log | tee gpurun_out/bench.json
LMOE_FUSED=0 timeout 300 python bench.py --no-cpu-baseline --no-extra 2>>gpurun_out/bench_err.log | tee gpurun_out/bench3.json
tail -3 gpurun_out/bench_err.log
