set -x
timeout 600 python -m pytest tests/test_gpu.py -x -q 2>&1 | tail -5
timeout 200 python scripts/diag_precision.py 2>&1 | grep TC
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -3
python scripts/prof_gemm.py 13 13 12 > gpurun_out/prof_plain.log 2>&1 && cat gpurun_out/prof_plain.log && \
ncu --set full --clock-control none --import-source on -k regex:cgemm -s 2 -c 1 -o gpurun_out/prof_cgemm2 python scripts/prof_gemm.py 13 13 12 > gpurun_out/ncu_cgemm2.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 1 --no-cpu-baseline 2>&1 | tail -1
