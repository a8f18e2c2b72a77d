# per-launch device times (ncu gpu__time_duration, one pass) of the GEMM kernels of one
# tensor-core step: bash scripts/time_pair_ncu.sh m n k [regex]
m=$1; n=$2; k=$3; re=${4:-cgemm}
python scripts/prof_gemm.py $m $n $k > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:$re --csv \
    python scripts/prof_gemm.py $m $n $k 2>/dev/null | grep -E "gpu__time_duration|cycles_elapsed" | awk -F'","' '{print $(NF-2), $NF}'
