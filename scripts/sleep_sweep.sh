for ns in 0 8 32 128 512; do
  for cfg in 1 2 3; do
    RKR_SLEEP_NS=$ns python bench.py --no-cpu-baseline --config $cfg --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('sleep $ns cfg $cfg fill_ms %.4f' % d['roofline']['fill_ms'])"
  done
done
