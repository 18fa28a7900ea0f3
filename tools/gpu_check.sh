#!/bin/bash
# quick GPU check: build, debug table, gpu tests, short bench; optional ncu of the output pass
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
timeout 300 python tools/dbg_lsm.py 2>&1 | tail -12
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -2
if [ "$1" = "prof" ]; then
  timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:lsm_output_pass -s 1 -c 1 \
     -o gpurun_out/prof_output python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/prof_output.log 2>&1
  timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:lsm_state_pass -s 1 -c 1 \
     -o gpurun_out/prof_state python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/prof_state.log 2>&1
fi
