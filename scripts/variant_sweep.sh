for v in 0 1 2 3; do
  for cfg in 2 3; do
    for R in 1 2; do
      RKR_VARIANT=$v RKR_R=$R python bench.py --no-cpu-baseline --config $cfg --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('variant $v cfg $cfg R $R fill_ms %.4f e2e_ms %.4f' % (d['roofline']['fill_ms'], d['e2e']['ms_per_step']))"
    done
  done
done
