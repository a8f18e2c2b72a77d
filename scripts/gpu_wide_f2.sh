# wide FFMA2 variant: parity tests, ncu device times FFMA vs FFMA2, pure-read HBM probe
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_fuzz.py -x -q -m gpu -k "wide or fuzz or degenerate" 2>&1 | tail -3
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/rbw scripts/probes/read_bw_probe.cu && timeout 300 /tmp/rbw
for shape in "5 26 3" "5 26 2" "4 25 4"; do
for v in 0 1 0 1; do
TN_WIDE_FFMA2=$v TN_PROF_PATH=wide ncu --metrics gpu__time_duration.sum --clock-control none -k regex:wide -c 2 --csv python scripts/prof_gemm.py $shape 2>/dev/null | grep wide | awk -F'","' -v g=$v '{print "f2=" g, $5, $(NF-2), $(NF-1), $NF}' | sed 's/(const.*long \*)//'
done
done
TN_PROF_PATH=wide ncu --set full --clock-control none --import-source on -k regex:wide -s 1 -c 1 -o gpurun_out/r02_wide_f2 -f python scripts/prof_gemm.py 5 26 3 > /dev/null 2>&1
echo ncu=$?
