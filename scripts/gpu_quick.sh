# tests + per-item traces + bench lines (no CPU leg) for configs 1-3
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for c in 1 2 3; do python scripts/trace_report.py --config $c; done
for c in 1 2 3; do python bench.py --no-cpu-baseline --config $c --steps 5 --warmup 3 | python -c "import json,sys; d=json.load(sys.stdin); print(d['config']['workload'][:8], 'fill_ms', round(d['roofline']['fill_ms'],4), 'solve_ms', round(d['ms_per_step'],4), 'e2e_ms', round(d['e2e']['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3))"; done
