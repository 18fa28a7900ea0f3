#!/bin/bash
# round-2 end check: full -m gpu suite, smoke, bench (both arms)
python -c "from paper_2503_05447_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1 || exit 1
rm -f gpurun_out/parity_errors.jsonl
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | grep -v "^  " | tail -4
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py 2>gpurun_out/bench_err.log > gpurun_out/bench_end.json; head -c 300 gpurun_out/bench_end.json; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 2>gpurun_out/bench_ref_err.log > gpurun_out/bench_ref_end.json; head -c 200 gpurun_out/bench_ref_end.json; echo
