# DMMA tail split (K-split clusters for the partial last wave): complex128 tests, per-launch
# times of configs[3], bench A/B (TN_DMMA_TAIL = 0 / 1, alternating)
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu.py -x -q -m gpu -k "complex128 or config3 or iqp or config0 or degenerate or lanes or dmma" 2>&1 | tail -3
for v in 0 1; do TN_DMMA_TAIL=$v timeout 300 python scripts/prof_dump.py 3 0 0.01 > gpurun_out/dump3_tail$v.log 2>&1; done
for v in 0 1 0 1; do
  TN_DMMA_TAIL=$v timeout 600 python bench.py --config 3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b3_tail$v.json 2> gpurun_out/b3_tail$v.err
  python -c "
import json; d=json.load(open('gpurun_out/b3_tail$v.json'))
print('tail=$v', round(d['ms_per_step'],3), 'ms/amp', round(d['amplitudes_per_s'],1), 'e2e', round(d['e2e']['value']/1e12,2), 'amp/s lanes', d['amplitudes_per_s_lanes']['value'] if d.get('amplitudes_per_s_lanes') else None, {k: (round(v['ms'],3), round(v.get('frac',0),3)) for k, v in d['kernels'].items()})"
done
