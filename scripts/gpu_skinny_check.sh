python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu.py -x -q -m gpu -k "skinny" 2>&1 | tail -2
TN_PROF_PATH=skinny bash scripts/time_pair_ncu.sh 4 3 26 skinny_kernel
