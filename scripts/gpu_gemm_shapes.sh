# the dominant GEMM shapes of configs 1 / 2 back to back under the power cap (K-chunks on/off)
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader -lms 500 > gpurun_out/clk_shapes.txt & P=$!
for s in "16 16 12 6" "16 15 14 6" "18 15 14 3" "16 16 12 6"; do
  timeout 600 python scripts/probes/gemm_b2b.py $s 2>&1 | tail -1
done
TN_GEMM_KCHUNK=0 timeout 600 python scripts/probes/gemm_b2b.py 16 15 14 6 2>&1 | tail -1 | sed 's/^/kchunk=0 /'
kill $P
