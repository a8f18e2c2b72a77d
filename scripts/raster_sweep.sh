# GEMM raster experiment: device time and DRAM bytes of the pair GEMM on one step shape for
# several TN_GEMM_GROUP_M values: bash scripts/raster_sweep.sh m n k "4 8 16"
m=$1; n=$2; k=$3
python scripts/prof_gemm.py $m $n $k > /dev/null 2>&1 || exit 1
for g in $4; do
  echo "group_m=$g"
  TN_GEMM_GROUP_M=$g ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,lts__t_sector_hit_rate.pct \
      --clock-control none -k regex:${RE:-cgemm2} -s 2 -c 1 --csv python scripts/prof_gemm.py $m $n $k 2>/dev/null \
      | grep -E "gpu__time|cycles_elapsed|dram__bytes|hit_rate" | awk -F'","' '{print "  ", $(NF-2), $(NF-1), $NF}'
done
