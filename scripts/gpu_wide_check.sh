python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu.py -x -q -m gpu -k "wide" 2>&1 | tail -2
TN_PROF_PATH=wide bash scripts/time_pair_ncu.sh 5 26 3 wide_kernel
TN_PROF_PATH=wide bash scripts/time_pair_ncu.sh 14 17 3 wide_kernel
