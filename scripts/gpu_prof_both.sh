# ncu --set full of the pair GEMM and the pack kernel on one config-1-like step (m=n=2^13, K=2^12)
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
python scripts/prof_gemm.py 13 13 12 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:cgemm2 -s 2 -c 1 -o gpurun_out/prof_cgemm -f python scripts/prof_gemm.py 13 13 12 > gpurun_out/ncu_cgemm.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pack_f16 -s 4 -c 2 -o gpurun_out/prof_pack -f python scripts/prof_gemm.py 13 13 12 > gpurun_out/ncu_pack.log 2>&1
echo ncu_rc=$?
