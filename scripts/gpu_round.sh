# Full measurement round: tests, bench lines (all configs), reference arms,
# ncu launch list of the default bench and ncu captures of the fill kernel.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()"
python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
python bench.py --config 1 > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
python bench.py --config 3 --steps 5 --warmup 3 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
python bench.py --config 4 --steps 5 --warmup 3 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
python bench.py --config 5 --steps 3 --warmup 3 > gpurun_out/bench_cfg5twin.json 2> gpurun_out/bench_cfg5twin.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_cfg2.json 2> gpurun_out/bench_ref_cfg2.err
python bench.py --impl reference --config 4 --steps 2 --warmup 1 > gpurun_out/bench_ref_cfg4.json 2> gpurun_out/bench_ref_cfg4.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:fill_persistent --csv --log-file gpurun_out/traffic_cfg3.csv python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:fill_persistent -s 4 -c 1 -o gpurun_out/prof_cfg2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:fill_persistent -s 4 -c 1 -o gpurun_out/prof_cfg3 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out
