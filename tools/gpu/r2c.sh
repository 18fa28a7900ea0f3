#!/bin/bash
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
rm -f gpurun_out/parity_errors.jsonl
timeout 900 python -m pytest tests/test_moe_gpu.py tests/test_lsm_gpu.py tests/test_nccl_gpu.py -x -q 2>&1 | grep -v "^  " | tail -8
timeout 300 python bench.py --no-cpu-baseline --no-extra 2>gpurun_out/bench_err.log | tee gpurun_out/bench.json | cut -c1-300
LMOE_TRACE=1 timeout 120 python tools/trace_lsm.py 2>&1 | tail -8
