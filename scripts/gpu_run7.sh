set -x
timeout 600 python -m pytest tests/test_gpu.py -x -q 2>&1 | tail -3
timeout 900 python bench.py --steps 3 --warmup 1 --no-cpu-baseline 2>&1 | tail -1
