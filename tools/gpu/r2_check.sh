#!/bin/bash
# one gpurun call: build, the GPU tests (parity log -> gpurun_out/parity_errors.jsonl), a short bench
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
rm -f gpurun_out/parity_errors.jsonl
timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} 2>&1 | grep -v "^  " | tail -15
timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS} 2>gpurun_out/bench_err.log | tee gpurun_out/bench.json
tail -3 gpurun_out/bench_err.log
