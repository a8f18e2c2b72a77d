# skinny v2 on K-blocked planar operands: parity (skinny + fuzz + bench-plan configs 2/4), device times, ncu --set full
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_fuzz.py -x -q -m gpu -k "skinny or fuzz or degenerate or slab" 2>&1 | tail -3
for shape in "4 3 26" "2 1 28" "4 2 26"; do
for r in 1 2; do
TN_PROF_PATH=skinny ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:skinny2 -c 2 --csv python scripts/prof_gemm.py $shape 2>/dev/null | grep -E "time_duration" | awk -F'","' -v s="$shape" '{print s, $(NF-2), $(NF-1), $NF}'
done
done
TN_PROF_PATH=skinny ncu --set full --clock-control none --import-source on -k regex:skinny2 -s 1 -c 1 -o gpurun_out/r02_skinny2_kb -f python scripts/prof_gemm.py 4 3 26 > /dev/null 2>&1
echo ncu=$?
TN_PROF_PATH=skinny ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:pack_planar -c 2 --csv python scripts/prof_gemm.py 4 3 26 2>/dev/null | grep -E "pack_planar" | awk -F'","' '{print "pack", $(NF-2), $(NF-1), $NF}'
