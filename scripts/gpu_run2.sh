set -x
timeout 300 python -m pytest tests/test_gpu.py -x -q -k "tensor_core or tc_matches or uses_tensor" 2>&1 | tail -15
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu.py -x -q -k "full_size" 2>&1 | tail -15
timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | tail -5
