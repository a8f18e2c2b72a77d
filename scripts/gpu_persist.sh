set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python -m pytest tests/test_gpu.py -x -q -k "tensor_core or slab or bounded or tc_matches" 2>&1 | tail -3
timeout 1200 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -3
python scripts/prof_dump.py 1 34 1.0 > gpurun_out/dump.log 2>&1
python scripts/prof_dump.py 2 33 1.0 > gpurun_out/dump_c2.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
