# round 2: build, GPU tests (optionally a -k filter), bench lines of the given configs
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests/ -x -v -m gpu --timeout 900 ${TEST_K:+-k "$TEST_K"} > gpurun_out/pytest.log 2>&1; grep -E "PASSED|FAILED|ERROR|Timeout" gpurun_out/pytest.log | tail -5; tail -3 gpurun_out/pytest.log
for c in ${BENCH_CONFIGS:-1}; do
  timeout 1200 python bench.py --config $c --steps ${STEPS:-3} --warmup 3 ${BENCH_ARGS} > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo rc=$?
  tail -3 gpurun_out/bench_c$c.err
done
