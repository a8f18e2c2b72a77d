# FFMA2 (packed fp32 pair FMA): throughput probe, skinny parity, skinny v2 FFMA vs FFMA2 device times, ncu --set full of FFMA2
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/ffma2_probe scripts/probes/ffma2_probe.cu && /tmp/ffma2_probe
timeout 900 python -m pytest tests/test_gpu.py -x -q -m gpu -k "skinny" 2>&1 | tail -3
for shape in "4 3 26" "2 1 28" "4 2 26"; do
for v in 0 1 0 1; do
TN_SKINNY_FFMA2=$v TN_PROF_PATH=skinny ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:skinny2 -c 3 --csv python scripts/prof_gemm.py $shape 2>/dev/null | grep -E "skinny" | awk -F'","' '{print $5, $(NF-2), $(NF-1), $NF}' | cut -c1-200
done
done
TN_PROF_PATH=skinny ncu --set full --clock-control none --import-source on -k regex:skinny2 -s 1 -c 1 -o gpurun_out/r02_skinny2_f2 -f python scripts/prof_gemm.py 4 3 26 > /dev/null 2>&1
echo ncu=$?
