set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu.py -x -q -k "skinny or wide" 2>&1 | tail -15
timeout 1500 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -5
python scripts/prof_dump.py 3 0 0.2 2>&1 | sed -n "/second run/,\$p"
python scripts/prof_dump.py 4 32 5 2>&1 | sed -n "/second run/,\$p" | grep -v gemm
