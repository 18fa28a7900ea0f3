#!/bin/bash
# full GPU suite with per-test durations (the suite's wall time is what the round-end run pays)
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
rm -f gpurun_out/parity_errors.jsonl
timeout 3000 python -m pytest tests -m gpu -q --durations=60 > gpurun_out/durations.txt 2>&1
tail -75 gpurun_out/durations.txt
