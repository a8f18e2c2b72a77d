# round 2: GPU tests + ncu --set full of the non-GEMM kernels (skinny, wide, planar pack,
# small, DMMA) on bench shapes; reports land in gpurun_out/r02_*.ncu-rep
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout ${TEST_TIMEOUT:-1200} python -m pytest tests/ -x -q -m gpu ${TEST_K:+-k "$TEST_K"} 2>&1 | tail -3
NCU="ncu --set full --clock-control none --import-source on"
TN_PROF_PATH=skinny python scripts/prof_gemm.py 4 3 26 && \
TN_PROF_PATH=skinny $NCU -k regex:skinny_kernel -s 1 -c 1 -o gpurun_out/r02_skinny -f python scripts/prof_gemm.py 4 3 26 > /dev/null 2>&1
TN_PROF_PATH=skinny $NCU -k regex:pack_planar -s 2 -c 1 -o gpurun_out/r02_pack_planar -f python scripts/prof_gemm.py 4 3 26 > /dev/null 2>&1
TN_PROF_PATH=wide python scripts/prof_gemm.py 5 26 3 && \
TN_PROF_PATH=wide $NCU -k regex:wide_kernel -s 1 -c 1 -o gpurun_out/r02_wide -f python scripts/prof_gemm.py 5 26 3 > /dev/null 2>&1
python scripts/run_config.py 3 2 && \
$NCU -k regex:zgemm -c 12 -o gpurun_out/r02_zgemm -f python scripts/run_config.py 3 1 > /dev/null 2>&1
$NCU -k regex:small_contract -c 12 -o gpurun_out/r02_small -f python scripts/run_config.py 3 1 > /dev/null 2>&1
echo done
