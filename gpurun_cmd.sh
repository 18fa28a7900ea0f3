python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
timeout 600 python -m pytest tests/test_moe_gpu.py -q -x 2>&1 | tail -25
