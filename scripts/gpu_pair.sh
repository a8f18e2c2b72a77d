set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 120 python -m pytest tests/test_gpu.py -x -q -k "tensor_core_path" 2>&1 | tail -5
timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -3
for s in "13 13 12" "14 14 10"; do timeout 60 python scripts/prof_gemm.py $s; TN_GEMM_PAIR=0 timeout 60 python scripts/prof_gemm.py $s; done
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
cat gpurun_out/bench.json | cut -c1-1200
