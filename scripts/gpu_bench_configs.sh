# bench lines of every config (1-GPU)
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
for c in 3 2 4 1; do
  timeout 1200 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo rc=$?
  cat gpurun_out/bench_c$c.json; tail -2 gpurun_out/bench_c$c.err
done
