# skinny v2 with the non-blocking producer: parity, device times by stage size; MMA-count probe of the pair GEMM
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu.py -x -q -m gpu -k "skinny" 2>&1 | tail -3
for shape in "4 3 26" "2 1 28" "4 2 26"; do
for ks in 256 128 256 128; do
TN_SK2_KS=$ks TN_PROF_PATH=skinny ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:skinny2 -c 2 --csv python scripts/prof_gemm.py $shape 2>/dev/null | grep -E "time_duration" | awk -F'","' -v k=$ks -v s="$shape" '{print s, "ks=" k, $(NF-2), $(NF-1), $NF}'
done
done
TN_PROF_PATH=skinny ncu --set full --clock-control none --import-source on -k regex:skinny2 -s 1 -c 1 -o gpurun_out/r02_skinny2_nb -f python scripts/prof_gemm.py 4 3 26 > /dev/null 2>&1
echo ncu=$?
# MMA-count sensitivity of the dominant pair GEMM under the power cap (timing only)
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader -lms 500 > gpurun_out/mma_probe_clk12.txt &
SMI=$!
python scripts/probes/mma_count_probe.py 8
kill $SMI
TN_NVCC_EXTRA=-DTN_PROBE_MMA9 python paper_2208_01498_b200/build.py -f > /dev/null || exit 1
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader -lms 500 > gpurun_out/mma_probe_clk9.txt &
SMI=$!
python scripts/probes/mma_count_probe.py 8
kill $SMI
python paper_2208_01498_b200/build.py -f > /dev/null
