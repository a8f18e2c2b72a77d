# raster group size A/B on the sliced configs (bench FLOP/s, GEMM frac, median clock)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for c in ${CONFIGS:-2 4}; do
  for G in ${GS:-4 2 8 4}; do
    TN_GEMM_GROUP_M=$G timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('config $c G=$G', '%.4g'%d['value'], 'gemm %.1f'%r['achieved'], 'clk', d['clocks']['sm_mhz'], 'W', d['clocks'].get('power_w'))"
  done
done
