set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import paper_2208_01498_b200 as t; print(t.lib.tn_version())"
timeout 300 python -m pytest tests/test_gpu.py -x -q -k "small_path or config0 or slic or iqp or sycamore or device or cdagger" 2>&1 | tail -15
timeout 240 python -m pytest tests/test_gpu.py -x -q -k "tensor_core_path" 2>&1 | tail -15
