# profiled CUDA graphs (bench.py's timed path) vs eager profiled launches: tests, configs[3]
# and configs[1] bench A/B (TN_PROFILE_GRAPH = 1 / 0)
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests/test_gpu_bench_plans.py tests/test_dist_gpu.py -x -q -m gpu -k "profiled or reuse or two_ranks or deferred" 2>&1 | tail -3
for v in 1 0 1 0; do
  TN_PROFILE_GRAPH=$v timeout 600 python bench.py --config 3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b3_pg$v.json 2> gpurun_out/b3_pg$v.err
  python -c "
import json; d=json.load(open('gpurun_out/b3_pg$v.json'))
print('c3 graph=$v', round(d['ms_per_step'],3), 'ms/amp', round(d['amplitudes_per_s'],1), 'check', d['check'], {k: round(v['ms']/20,4) for k, v in d['kernels'].items()})"
done
for v in 1 0; do
  TN_PROFILE_GRAPH=$v timeout 900 python bench.py --config 1 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/b1_pg$v.json 2> gpurun_out/b1_pg$v.err
  python -c "
import json; d=json.load(open('gpurun_out/b1_pg$v.json'))
print('c1 graph=$v', round(d['value']/1e12,1), round(d['ms_per_step'],1), d['amplitudes_per_s'], d['roofline']['frac'], d['check'], d['gpu_launches'])"
done
