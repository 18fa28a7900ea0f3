python -c "from paper_2503_05447_b200 import _build; _build.build()" || exit 1
INST=mamba2 LMOE_TRACE=1 LMOE_OP_ORDER=1 timeout 120 python tools/trace_lsm.py 2>&1 | tail -3
for o in 0 1; do LMOE_OP_ORDER=$o timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('order', $o, d['value']/1e6, d['roofline']['frac'], d['phase_ms_per_step'])"; done
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
