# the driver's round-end checks: build, the whole GPU suite, smoke
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 2400 python -m pytest tests/ -x -q -m gpu --timeout 900 > gpurun_out/pytest_tests_final.log 2>&1; tail -3 gpurun_out/pytest_tests_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
