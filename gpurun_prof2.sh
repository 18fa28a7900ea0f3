#!/bin/bash
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
export PYTHONPATH=.
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:lsm_vec_bwd_chunk -c 1 \
   -o gpurun_out/prof_vec_bwd_chunk python tools/bwd_vec_time.py once 65536 gla > gpurun_out/prof_vbc.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:lsm_output_pass_vec -c 1 \
   -o gpurun_out/prof_vec_out python tools/bwd_vec_time.py t 65536 gla > gpurun_out/prof_vo.log 2>&1
