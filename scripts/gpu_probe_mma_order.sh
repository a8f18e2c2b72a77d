# MMA issue order of the pair kernel (operand toggling vs power): (16, 16, 12) back to back,
# with a temporary `#if TN_MMA_ORDER` in mma_loop_pair (removed after the measurement): 0 =
# re.re, -im.im, re.im, im.re (kept); 1 = re.re, re.im, im.re, -im.im (A kept for two MMAs)
set -x
for v in 0 1; do
  TN_NVCC_EXTRA=-DTN_MMA_ORDER=$v python -c "import sys; sys.path.insert(0,'paper_2208_01498_b200'); import build; build.build(force=True)" || exit 1
  cp paper_2208_01498_b200/libtn_b200.so /tmp/lib_o$v.so
done
for v in 0 1 0 1 0 1; do
  cp /tmp/lib_o$v.so paper_2208_01498_b200/libtn_b200.so
  timeout 300 python scripts/probes/gemm_b2b.py 16 16 12 10 2>&1 | tail -1 | sed "s/^/order=$v /"
done
