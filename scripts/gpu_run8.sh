set -x
timeout 600 python -m pytest tests/test_gpu.py -x -q -k "dmma or small_path or config0 or iqp" 2>&1 | tail -3
timeout 600 python scripts/run_config.py 3 16 2>&1 | tail -3
timeout 300 python scripts/run_config.py 0 16 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "config3" 2>&1 | tail -3
