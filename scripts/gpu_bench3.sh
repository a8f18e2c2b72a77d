set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
for c in 1 2 4; do timeout 1500 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bc$c.json 2> gpurun_out/bc$c.err; echo rc=$?; done
