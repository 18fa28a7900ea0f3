#!/bin/bash
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
export PYTHONPATH=.
timeout 900 python -m pytest tests/test_moe_gpu.py tests/test_model_gpu.py -q 2>&1 | tail -3
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('layer', d['layer']['ms_per_step'], d['layer']['roofline']['frac'])"
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:moe_gemm python tools/block_once.py 2>&1 | grep -E "moe_gemm|gpu__time|tensor" | tail -12
