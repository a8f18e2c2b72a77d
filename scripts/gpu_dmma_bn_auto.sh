# DMMA 64 x 32 tiles for steps under one wave of 64 x 64 tiles (auto) vs never (TN_DMMA_BN=64)
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu.py -x -q -m gpu -k "complex128 or config3 or iqp or lanes or dmma" 2>&1 | tail -2
for v in 0 64; do TN_DMMA_BN=$v timeout 300 python scripts/prof_dump.py 3 0 0.01 2>&1 | awk '/-- second run --/{f=1} f' | grep dmma | sed "s/^/bn=$v /"; done
for v in 0 64 0 64; do
  TN_DMMA_BN=$v timeout 600 python bench.py --config 3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b3_bn$v.json 2> gpurun_out/b3_bn$v.err
  python -c "
import json; d=json.load(open('gpurun_out/b3_bn$v.json'))
print('bn=$v', round(d['ms_per_step'],3), 'ms/amp', round(d['amplitudes_per_s'],1), 'dmma', round(d['kernels']['zgemm_dmma_kernel']['ms']/20,4), round(d['kernels']['zgemm_dmma_kernel']['frac'],3), 'skinny', round(d['kernels']['skinny_kernel']['ms']/20,4))"
done
