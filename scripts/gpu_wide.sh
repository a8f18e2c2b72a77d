# wide kernel: tests, configs[3] bench (gathered wide on / off), ncu time of the (5,26,3) c64 step
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_bench_plans.py -x -q -m gpu -k "wide or config3 or iqp or degenerate or config0 or lanes or reuse or profiled" 2>&1 | tail -2
for v in 1 0 1 0; do
TN_WIDE_GATHER=$v timeout 600 python bench.py --config 3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b3_w$v.json 2> gpurun_out/b3_w$v.err
python -c "
import json; d=json.load(open('gpurun_out/b3_w$v.json'))
print('gather=$v', round(d['ms_per_step'],3), 'ms/amp', round(d['amplitudes_per_s'],1), 'amp/s; lanes', round(d['amplitudes_per_s_lanes']['value'],1), {k: (round(v['ms']/20,3), round(v.get('frac',0),3)) for k, v in d['kernels'].items()})"
done
for v in 1 0; do
TN_WIDE_GATHER=$v TN_PROF_PATH=wide ncu --metrics gpu__time_duration.sum --clock-control none -k regex:wide -c 2 --csv python scripts/prof_gemm.py 5 26 3 2>/dev/null | grep wide | awk -F'","' -v g=$v '{print "gather=" g, $(NF-2), $(NF-1), $NF}'
done
