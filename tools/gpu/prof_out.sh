#!/bin/bash
# one ncu --set full capture of the output pass at the bench shape (read here with tools/ncu_summary.py)
python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
timeout 600 python -m pytest tests/test_nccl_gpu.py -x -q 2>&1 | tail -3
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"^lsm_output_pass\$|lsm_output_pass<" -s 1 -c 1 \
   -o gpurun_out/prof_out python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extra --e2e-steps 1 > gpurun_out/prof_out.log 2>&1
ls -la gpurun_out
