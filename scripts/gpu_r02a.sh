# Round 2, first GPU pass: the full GPU suite (incl. the reference-golden
# full-size tests), smoke, the default bench (config 3) and its reference arm,
# and one ncu --set full capture of the config-3 fill.  Output: gpurun_out/r02a/.
O=gpurun_out/r02a
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x --durations=15 > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 900 python bench.py --impl reference > $O/bench_ref_cfg3.json 2> $O/bench_ref_cfg3.err
timeout 600 python bench.py --config 2 --no-ncu > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fill_ -s 3 -c 1 -o $O/prof_cfg3 -f python bench.py --ncu-probe --config 3 > $O/ncu_full.log 2>&1
ls -la $O
