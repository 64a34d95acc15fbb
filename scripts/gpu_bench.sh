set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
python bench.py --config 3 --steps 5 --warmup 3 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
python bench.py --config 1 > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 3 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:fill_persistent --csv --log-file gpurun_out/traffic_cfg3.csv python bench.py --config 3 --steps 1 --warmup 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:fill_persistent -s 2 -c 1 -o gpurun_out/prof_cfg3 python bench.py --config 3 --steps 1 --warmup 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:fill_persistent -s 2 -c 1 -o gpurun_out/prof_cfg2 python bench.py --steps 1 --warmup 3 > /dev/null 2>&1
ls -la gpurun_out
