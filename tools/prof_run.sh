#!/bin/bash
# ncu captures for the LSM kernels (run under gpurun).  Never used for bench numbers.
set -x
python -m paper_2503_05447_b200._build >/dev/null 2>&1
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/launches_bench.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:lsm_output_pass -s 1 -c 1 \
   -o gpurun_out/prof_output python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/prof_output.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:lsm_state_pass -s 1 -c 1 \
   -o gpurun_out/prof_state python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/prof_state.log 2>&1
ls -la gpurun_out
