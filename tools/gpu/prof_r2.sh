#!/bin/bash
# ncu evidence for profiles/ (never bench numbers): launch lists + full captures of the hot kernels
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
NCU=/usr/local/cuda/bin/ncu
export PYTHONPATH=.
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 $NCU --metrics $M --clock-control none --csv --log-file gpurun_out/r2_bench_launches.csv \
   python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extra --e2e-steps 1 > /dev/null 2>&1
timeout 600 $NCU --metrics $M --clock-control none --csv --log-file gpurun_out/r2_mamba_bwd_launches.csv \
   python tools/bwd_once.py > /dev/null 2>&1
for k in lsm_output_pass lsm_state_pass; do
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"^$k\$|$k<" -s 1 -c 1 \
     -o gpurun_out/r2_prof_$k python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extra --e2e-steps 1 > /dev/null 2>&1
done
ls -la gpurun_out
