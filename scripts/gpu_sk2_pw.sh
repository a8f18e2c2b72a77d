# skinny v2 with a dedicated producer warp (default; TN_SK2_PW=0: lane 0 of consumer warp 0) -- parity, device times (ncu)
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 1200 python -m pytest tests/test_gpu.py tests/test_gpu_fuzz.py -x -q -m gpu -k "skinny or slab or fuzz or degenerate or config" 2>&1 | tail -2
for shape in "4 3 26" "4 2 26" "2 1 28" "0 0 30" "3 3 26" "2 2 27"; do
for pw in 0 1 0 1; do
TN_SK2_PW=$pw TN_PROF_PATH=skinny timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:skinny2 -c 2 --csv python scripts/prof_gemm.py $shape 2>/dev/null | grep -E "time_duration" | awk -F'","' -v s="$shape" -v b=$pw '{print s, "pw=" b, $(NF-2), $(NF-1), $NF}'
done
done
