# skinny v2: tests, ncu device times of v1 vs v2 on the (4,3,26) shape, ncu --set full of v2
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu.py -x -q -m gpu -k "skinny" 2>&1 | tail -3
for v in 0 1; do
TN_SKINNY_V2=$v TN_PROF_PATH=skinny ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:skinny -c 3 --csv python scripts/prof_gemm.py ${SHAPE:-4 3 26} 2>/dev/null | grep -E "skinny" | awk -F'","' '{print $5, $(NF-2), $(NF-1), $NF}' | cut -c1-200
done
TN_PROF_PATH=skinny ncu --set full --clock-control none --import-source on -k regex:skinny2 -s 1 -c 1 -o gpurun_out/r02_skinny2 -f python scripts/prof_gemm.py ${SHAPE:-4 3 26} > /dev/null 2>&1
echo ncu=$?
