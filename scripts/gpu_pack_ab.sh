# fp16x2 pack A/B (a temporary TN_PACK_MINB macro, removed after): 4 CTAs per SM (64 registers,
# spills) vs 3 (80, no spills), one scale multiply in both; configs[1] bench pack share, alternating
for v in 4 3; do
  TN_NVCC_EXTRA=-DTN_PACK_MINB=$v python -c "import sys; sys.path.insert(0,'paper_2208_01498_b200'); import build; build.build(force=True)" || exit 1
  cp paper_2208_01498_b200/libtn_b200.so /tmp/lib_pk$v.so
done
for v in 4 3 4 3; do
  cp /tmp/lib_pk$v.so paper_2208_01498_b200/libtn_b200.so
  timeout 900 python bench.py --config 1 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/b1_pk$v.json 2> gpurun_out/b1_pk$v.err
  python -c "
import json; d=json.load(open('gpurun_out/b1_pk$v.json'))
print('minb=$v', round(d['value']/1e12,1), d['clocks']['sm_mhz'], {k: (round(v['ms'],1), round(v['share_of_step'],4), round(v.get('frac',0),3)) for k, v in d['kernels'].items() if v['ms'] > 1})"
done
