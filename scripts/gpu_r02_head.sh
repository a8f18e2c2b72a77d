# re-entry check of HEAD: GPU tests, smoke, default bench, configs[3] bench
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 2400 python -m pytest tests/ -x -v -m gpu --timeout 900 > gpurun_out/pytest_head.log 2>&1; tail -3 gpurun_out/pytest_head.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1800 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_head_c1.json 2> gpurun_out/bench_head_c1.err; echo c1=$?
timeout 900 python bench.py --config 3 --steps 20 --warmup 5 > gpurun_out/bench_head_c3.json 2> gpurun_out/bench_head_c3.err; echo c3=$?
