# re-entry session 4: build, whole GPU suite, smoke, default bench line
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 2400 python -m pytest tests/ -x -q -m gpu --timeout 900 > gpurun_out/pytest_reentry4.log 2>&1; tail -5 gpurun_out/pytest_reentry4.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_reentry4.json 2> gpurun_out/bench_reentry4.err; echo bench_rc=$?
cat gpurun_out/bench_reentry4.json; tail -3 gpurun_out/bench_reentry4.err
# the reference arm, as the driver launches it
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference_reentry4.json 2> gpurun_out/bench_reference_reentry4.err; echo ref_rc=$?
tail -c 600 gpurun_out/bench_reference_reentry4.json
