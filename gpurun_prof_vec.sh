#!/bin/bash
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
export PYTHONPATH=.
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/vec_launches.csv python tools/bwd_vec_time.py once 262144 gla > gpurun_out/vec_launches.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:lsm_vec_bwd_chunk -s 2 -c 1 \
   -o gpurun_out/prof_vec_bwd_chunk python tools/bwd_vec_time.py once 65536 gla > gpurun_out/prof_vbc.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:lsm_output_pass_vec -s 1 -c 1 \
   -o gpurun_out/prof_vec_out python tools/bwd_vec_time.py once 65536 gla > gpurun_out/prof_vo.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:lsm_vec_carry -s 1 -c 1 \
   -o gpurun_out/prof_vec_carry python tools/bwd_vec_time.py once 65536 gla > gpurun_out/prof_vc.log 2>&1
ls -la gpurun_out
