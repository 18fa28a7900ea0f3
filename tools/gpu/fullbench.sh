#!/bin/bash
# the driver's round-end sequence: build, default bench, reference arm
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
timeout 1200 python bench.py 2>gpurun_out/bench_err.log | tee gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 2>gpurun_out/bench_ref_err.log | tee gpurun_out/bench_ref.json
tail -5 gpurun_out/bench_err.log; tail -3 gpurun_out/bench_ref_err.log
