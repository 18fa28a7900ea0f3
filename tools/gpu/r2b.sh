#!/bin/bash
# build, the new/changed-path tests first (fail fast), a short bench, then the whole GPU suite
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
make -s -C oracle
rm -f gpurun_out/parity_errors.jsonl
timeout 900 python -m pytest tests/test_nccl_gpu.py tests/test_tensor_bridge_gpu.py tests/test_lsm_gpu.py -x -q 2>&1 | grep -v "^  " | tail -15
timeout 300 python bench.py --no-cpu-baseline --no-extra 2>gpurun_out/bench_err.log | tee gpurun_out/bench.json
LMOE_TRACE=1 timeout 120 python tools/trace_lsm.py 2>&1 | tail -16
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | grep -v "^  " | tail -15
