#!/bin/bash
# ncu evidence for profiles/ (run under gpurun).  Never used for bench numbers.
#   launch list of the bench command (per-kernel durations, cold and serialised) and one
#   --set full capture of each hot kernel
python -m paper_2503_05447_b200._build >/dev/null 2>&1
NCU=/usr/local/cuda/bin/ncu
export PYTHONPATH=.
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extra --e2e-steps 1 > gpurun_out/launches_bench.log 2>&1
for k in lsm_output_pass lsm_state_pass; do
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"^$k\$|$k<" -s 1 -c 1 \
     -o gpurun_out/prof_$k python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extra --e2e-steps 1 > gpurun_out/prof_$k.log 2>&1
done
# TokenVector (GLA) forward and backward kernels, cfg3 shape
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/gla_launches.csv python tools/bwd_vec_time.py once 262144 gla > gpurun_out/gla_launches.log 2>&1
for k in lsm_output_pass_vec lsm_vec_bwd_chunk lsm_vec_carry; do
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$k -c 1 \
     -o gpurun_out/prof_$k python tools/bwd_vec_time.py once 262144 gla > gpurun_out/prof_$k.log 2>&1
done
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:lsm_mamba_dgate -s 1 -c 1 \
   -o gpurun_out/prof_dgate python tools/bwd_once.py > gpurun_out/prof_dgate.log 2>&1
ls -la gpurun_out
