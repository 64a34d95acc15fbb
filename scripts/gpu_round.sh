# Full measurement round: tests, smoke, bench lines (all configs), reference
# arms, the ncu launch list of the default bench, full captures of the fill
# kernels, per-step traces, sanitizers.  Output: gpurun_out/round/.
#   gpurun --timeout 3600 -- 'bash scripts/gpu_round.sh'
O=gpurun_out/round
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu --durations=15 > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
# the default bench (config 3: live L2 probe + ncu counter pass + CPU baseline) and its reference arm
timeout 900 python bench.py > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 900 python bench.py --impl reference > $O/bench_ref_cfg3.json 2> $O/bench_ref_cfg3.err
for c in 1 2; do timeout 600 python bench.py --config $c > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; done
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 600 python bench.py --config 5 --steps 3 --warmup 3 > $O/bench_cfg5twin.json 2> $O/bench_cfg5twin.err
timeout 600 python bench.py --impl reference --config 2 --steps 3 --warmup 1 > $O/bench_ref_cfg2.json 2> $O/bench_ref_cfg2.err
timeout 600 python bench.py --impl reference --config 4 --steps 2 --warmup 1 > $O/bench_ref_cfg4.json 2> $O/bench_ref_cfg4.err
# launch list of the default bench (per-launch times, cold caches, serialised)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_cfg3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ncu > /dev/null 2>&1
# full captures of the fill kernel: config 3 (headline) and config 2
for c in 3 2; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fill_tiles -s 3 -c 1 -o $O/prof_cfg$c -f python bench.py --ncu-probe --config $c > $O/ncu_cfg$c.log 2>&1
done
for c in 3 2; do timeout 300 python scripts/trace_tiles.py --config $c > $O/trace_cfg$c.txt 2>&1; done
for tool in memcheck racecheck synccheck; do
timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py > $O/sanitize_$tool.txt 2>&1; echo "rc=$?" >> $O/sanitize_$tool.txt
done
ls -la $O
