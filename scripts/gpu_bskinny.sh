# gathered batched skinny kernel + CTA-per-output reduction: skinny / complex128 / plan tests,
# configs[3] per-launch times and bench A/B (TN_SKINNY_GATHER = 1 / 0)
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests/test_gpu.py tests/test_gpu_fuzz.py -x -q -m gpu -k "skinny or complex128 or config3 or iqp or config0 or degenerate or lanes or random" 2>&1 | tail -3
timeout 300 python scripts/prof_dump.py 3 0 0.01 > gpurun_out/dump3_bs.log 2>&1
for v in 1 0 1 0; do
  TN_SKINNY_GATHER=$v timeout 600 python bench.py --config 3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b3_bs$v.json 2> gpurun_out/b3_bs$v.err
  python -c "
import json; d=json.load(open('gpurun_out/b3_bs$v.json'))
print('gather=$v', round(d['ms_per_step'],3), 'ms/amp', round(d['amplitudes_per_s'],1), 'e2e', round(d['e2e']['value']/1e12,2), 'lanes', d['amplitudes_per_s_lanes']['value'] if d.get('amplitudes_per_s_lanes') else None, {k: (round(v['ms'],3), round(v.get('frac',0),3)) for k, v in d['kernels'].items()})"
done
