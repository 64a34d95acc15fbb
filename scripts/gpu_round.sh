# Full measurement round: tests, bench lines (all configs), reference arms,
# ncu launch list of the default bench, DRAM traffic and full captures of the
# fill kernels.  Output: gpurun_out/round/.
set -x
O=gpurun_out/round
mkdir -p $O
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()"
python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
python bench.py --config 1 > $O/bench_cfg1.json 2> $O/bench_cfg1.err
python bench.py --config 3 --steps 5 --warmup 3 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
python bench.py --config 4 --steps 5 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
python bench.py --config 5 --steps 3 --warmup 3 > $O/bench_cfg5twin.json 2> $O/bench_cfg5twin.err
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_cfg2.json 2> $O/bench_ref_cfg2.err
python bench.py --impl reference --config 4 --steps 2 --warmup 1 > $O/bench_ref_cfg4.json 2> $O/bench_ref_cfg4.err
# launch list of the default bench (per-launch times, cold caches, serialised)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
# DRAM traffic of one fill launch per config
for c in 2 3; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k regex:fill_tiles -s 3 -c 1 --csv --log-file $O/traffic_cfg$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k regex:fill_tiles -s 3 -c 1 --csv --log-file $O/traffic_cfg4.csv python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
# full captures of the fill kernel (config 2 headline, config 3 largest)
for c in 2 3; do
ncu --set full --clock-control none --import-source on -k regex:fill_tiles -s 3 -c 1 -o $O/prof_cfg$c -f python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
for c in 1 2 3; do python scripts/trace_tiles.py --config $c > $O/trace_cfg$c.txt 2>&1; done
ls -la $O
