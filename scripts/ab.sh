# A/B: bench fill/solve times and per-item traces for two builds of librkr.so.
#   bash scripts/ab.sh abtest/librkr_old.so paper_2307_01236_b200/librkr.so [configs]
mkdir -p gpurun_out
CFGS=${3:-"1 2 3"}
for lib in "$1" "$2"; do
  for c in $CFGS; do
    echo "== $lib config $c"
    RKR_LIB=$PWD/$lib python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d.get('roofline',{}); print('solve_ms %.4f fill_ms %.4f e2e_ms %.4f frac %.3f' % (d['ms_per_step'], r.get('fill_ms',0), d['e2e'].get('ms_per_step',0), r.get('frac',0)))
    else: print(l.rstrip())"
    RKR_LIB=$PWD/$lib python scripts/trace_report.py --config $c
  done
done
