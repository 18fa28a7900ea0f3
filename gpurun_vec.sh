#!/bin/bash
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -25
PYTHONPATH=. timeout 300 python tools/bwd_vec_time.py 2>&1 | tail -5
PYTHONPATH=. timeout 300 python tools/bwd_vec_time.py t 262144 hgrn2 2>&1 | tail -5
NCU=/usr/local/cuda/bin/ncu
PYTHONPATH=. timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/vec_launches.csv python tools/bwd_vec_time.py once 262144 gla > gpurun_out/vec_launches.log 2>&1
