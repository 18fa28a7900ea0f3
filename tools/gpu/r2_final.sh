#!/bin/bash
# round-2 end-state check: gpu tests, smoke, bench (both arms), ncu evidence of the bench step
python -c "from paper_2503_05447_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1 || exit 1
rm -f gpurun_out/parity_errors.jsonl
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | grep -v "^  " | tail -8
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py 2>gpurun_out/bench_err.log > gpurun_out/bench.json; head -c 600 gpurun_out/bench.json; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 2>gpurun_out/bench_ref_err.log > gpurun_out/bench_ref.json; head -c 200 gpurun_out/bench_ref.json; echo
NCU=/usr/local/cuda/bin/ncu
export PYTHONPATH=.
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 $NCU --metrics $M --clock-control none --csv --log-file gpurun_out/r2_local_bench_launches.csv \
   python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extra --e2e-steps 1 > /dev/null 2>&1
timeout 600 $NCU --metrics $M --clock-control none --csv --log-file gpurun_out/r2_mamba_bwd_launches2.csv \
   python tools/bwd_once.py > /dev/null 2>&1
for k in lsm_output_pass lsm_local_fix; do
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"^$k\$|$k<" -s 1 -c 1 \
     -o gpurun_out/r2_local_prof_$k python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extra --e2e-steps 1 > /dev/null 2>&1
done
ls -la gpurun_out
