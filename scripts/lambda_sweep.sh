mkdir -p gpurun_out
for cfg in 3 2 1; do
for R in 1 2; do
for lam in 1 2 4 8 16 32 64; do
  RKR_R=$R RKR_LAMBDA=$lam python bench.py --no-cpu-baseline --config $cfg --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('cfg $cfg R $R lam $lam fill_ms %.3f solve_ms %.3f' % (d['roofline']['fill_ms'], d['ms_per_step']))"
done; done; done
