#!/bin/bash
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
export PYTHONPATH=.
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"lsm_output_pass_vec|lsm_state_pass_vec" -c 2 \
   -o gpurun_out/prof_vec_fwd python tools/bwd_vec_time.py t 65536 gla > gpurun_out/prof_vf.log 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/vec_launches.csv python tools/bwd_vec_time.py once 262144 gla > gpurun_out/vec_launches.log 2>&1
