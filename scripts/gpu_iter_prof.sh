# tests + bench + one ncu capture of the GEMM
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -5
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
python scripts/prof_gemm.py 13 13 12 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:cgemm -s 2 -c 1 -o gpurun_out/prof_cgemm -f python scripts/prof_gemm.py 13 13 12 > gpurun_out/ncu_cgemm.log 2>&1
echo ncu_rc=$?
