# the bench plan's dominant tensor-core GEMM: DRAM bytes per launch vs raster group size,
# and one ncu --set full capture (profiles/r02 traffic) -- shape from the plan summary
set -x
python scripts/plan_summary.py 1 ${TGT:-32} > gpurun_out/plan_c1.log 2>&1
SHAPE=$(grep -m1 "tc nb,m,n,k" gpurun_out/plan_c1.log | sed 's/.*= (\([0-9]*\), \([0-9]*\), \([0-9]*\), \([0-9]*\)).*/\2 \3 \4 \1/')
echo "dominant shape (m n k nb): $SHAPE"
for G in ${GROUPS_M:-4 8 16}; do
  for S in 1 0; do
    TN_GEMM_GROUP_M=$G TN_GEMM_SERP=$S ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:cgemm2 -c 1 --csv python scripts/prof_gemm.py $SHAPE 2>/dev/null | grep -E "dram__bytes|duration|per_second" | awk -F'","' -v g=$G -v s=$S '{print "G=" g " serp=" s, $(NF-2), $(NF-1), $NF}'
  done
done
[ -n "$NO_FULL" ] || ncu --set full --clock-control none --import-source on -k regex:cgemm2 -c 1 -o gpurun_out/r02_gemm_dominant -f python scripts/prof_gemm.py $SHAPE > /dev/null 2>&1
echo ncu=$?
