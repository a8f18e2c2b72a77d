# K-chunk length sweep on K = 16384 pair GEMMs under the power cap (a temporary
# TN_GEMM_KCHUNK_STAGES override in finish_tc_shape, removed after: no setting stood out)
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
for rep in 1 2; do
  for cs in 128 256 512 100000; do
    TN_GEMM_KCHUNK_STAGES=$cs timeout 600 python scripts/probes/gemm_b2b.py 16 15 14 5 2>&1 | tail -1 | sed "s/^/cs=$cs /"
  done
done
for cs in 128 256 512; do
  TN_GEMM_KCHUNK_STAGES=$cs timeout 600 python scripts/probes/gemm_b2b.py 16 12 16 4 2>&1 | tail -1 | sed "s/^/cs=$cs /"
done
