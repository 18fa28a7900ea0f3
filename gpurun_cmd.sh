python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
timeout 600 python -m pytest tests/test_moe_gpu.py -q -x 2>&1 | tail -3
timeout 300 python tools/bench_moe.py
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/moe_launches.csv env STEPS=1 python tools/bench_moe.py > /dev/null 2>&1
