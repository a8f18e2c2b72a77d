# one-tile-per-pair vs persistent pair kernel on long-K steps (ncu device time)
python -c "import __graft_entry__ as g; g.build()" || exit 1
for shape in "18 12 12" "16 16 12" "19 9 13"; do
  echo "shape $shape default"; bash scripts/time_pair_ncu.sh $shape cgemm2
  echo "shape $shape persistent"; TN_GEMM_GROUP_M=4 TN_PERSIST_MAX_STAGES=100000 bash scripts/time_pair_ncu.sh $shape cgemm2
done
