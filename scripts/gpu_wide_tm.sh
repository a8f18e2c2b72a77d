# complex128 wide tile rows: 64 (TN_WD_TM_C128 default) vs 32 (round-2 kernel), configs[3] bench A/B
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu.py -x -q -m gpu -k "wide or config3 or iqp or lanes" 2>&1 | tail -2
cp paper_2208_01498_b200/libtn_b200.so /tmp/lib_tm64.so
TN_NVCC_EXTRA=-DTN_WD_TM_C128=32 python -c "import sys; sys.path.insert(0,'paper_2208_01498_b200'); import build; build.build(force=True)" || exit 1
cp paper_2208_01498_b200/libtn_b200.so /tmp/lib_tm32.so
for v in 64 32 64 32; do
  cp /tmp/lib_tm$v.so paper_2208_01498_b200/libtn_b200.so
  timeout 600 python bench.py --config 3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b3_tm$v.json 2> gpurun_out/b3_tm$v.err
  python -c "
import json; d=json.load(open('gpurun_out/b3_tm$v.json'))
print('tm=$v', round(d['ms_per_step'],3), 'ms/amp', round(d['amplitudes_per_s'],1), 'lanes', round(d['amplitudes_per_s_lanes']['value'],1), 'wide', round(d['kernels']['wide_kernel']['ms']/20, 4), round(d['kernels']['wide_kernel']['frac'],3))"
done
cp /tmp/lib_tm64.so paper_2208_01498_b200/libtn_b200.so
