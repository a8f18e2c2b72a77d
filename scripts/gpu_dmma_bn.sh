# DMMA gather N-tile width A/B on configs[3]: TN_DMMA_BN = 64 / 32 / auto
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu.py -x -q -m gpu -k "complex128 or config3 or iqp or config0 or dmma" 2>&1 | tail -2
for v in 64 32 0 64 32 0; do
  TN_DMMA_BN=$v timeout 600 python bench.py --config 3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b3_bn$v.json 2> gpurun_out/b3_bn$v.err
  python -c "
import json; d=json.load(open('gpurun_out/b3_bn$v.json'))
print('bn=$v', round(d['ms_per_step'],3), 'ms/amp', round(d['amplitudes_per_s'],1), 'amp/s; lanes', round(d['amplitudes_per_s_lanes']['value'],1), 'dmma ms', round(d['kernels']['zgemm_dmma_kernel']['ms'],3))"
done
