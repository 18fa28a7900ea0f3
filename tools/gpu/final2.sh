#!/bin/bash
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
rm -f gpurun_out/parity_errors.jsonl
timeout 900 python -m pytest tests/test_sp_gpu.py tests/test_local_gpu.py tests/test_model_gpu.py tests/test_determinism_gpu.py -q -x 2>&1 | grep -v "^  " | tail -8
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | grep -v "^  " | tail -8
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py 2>gpurun_out/bench_err.log > gpurun_out/bench.json; head -c 400 gpurun_out/bench.json; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 2>gpurun_out/bench_ref_err.log > gpurun_out/bench_ref.json; head -c 200 gpurun_out/bench_ref.json; echo
