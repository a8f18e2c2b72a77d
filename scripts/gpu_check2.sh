set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -3
for c in 1 4 2; do timeout 1200 python bench.py --config $c --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/bc$c.json 2> gpurun_out/bc$c.err; echo rc=$?; done
