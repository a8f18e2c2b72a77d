# L2->SM traffic vs power-capped GEMM time: the (16, 16, 12) pair step back to back with the
# normal library, then with A loaded on even stages only after every ring slot was filled once
# (an #ifdef TN_PROBE_HALF_A in the pair kernel's producer, removed after the measurement: a
# third less L2->SM traffic, wrong results), alternating
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
cp paper_2208_01498_b200/libtn_b200.so /tmp/lib_normal.so
TN_NVCC_EXTRA=-DTN_PROBE_HALF_A python -c "import sys; sys.path.insert(0,'paper_2208_01498_b200'); import build; build.build(force=True)" || exit 1
cp paper_2208_01498_b200/libtn_b200.so /tmp/lib_halfa.so
for v in normal halfa normal halfa; do
  cp /tmp/lib_$v.so paper_2208_01498_b200/libtn_b200.so
  nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader -lms 500 > gpurun_out/clk_$v.txt & P=$!
  timeout 300 python scripts/probes/mma_count_probe.py 12 2>&1 | tail -1 | sed "s/^/$v: /"
  kill $P; sort -n gpurun_out/clk_$v.txt | awk -F, '{print $1}' | sort -n | awk '{a[NR]=$1} END {print "median sm clock", a[int(NR/2)]}'
done
