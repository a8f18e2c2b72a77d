set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -3
python scripts/prof_dump.py 1 34 1.0 > gpurun_out/dump.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
cat gpurun_out/bench.json | cut -c1-1500
