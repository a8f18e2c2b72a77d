# small waves with a CTA -> step table; wide one-CTA-per-tile grid A/B (TN_WIDE_FULLGRID)
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests/test_gpu.py tests/test_gpu_fuzz.py -x -q -m gpu -k "small or wide or config0 or config3 or iqp or degenerate or random or lanes" 2>&1 | tail -2
for v in 0 1 0 1; do
  TN_WIDE_FULLGRID=$v timeout 600 python bench.py --config 3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b3_fg$v.json 2> gpurun_out/b3_fg$v.err
  python -c "
import json; d=json.load(open('gpurun_out/b3_fg$v.json'))
print('fullgrid=$v', round(d['ms_per_step'],3), 'ms/amp', round(d['amplitudes_per_s'],1), {k: round(v['ms']/20,4) for k, v in d['kernels'].items()})"
done
for v in 0 1; do TN_WIDE_FULLGRID=$v TN_PROF_PATH=wide ncu --metrics gpu__time_duration.sum --clock-control none -k regex:wide -c 2 --csv python scripts/prof_gemm.py 5 26 3 2>/dev/null | grep wide | awk -F'","' -v g=$v '{print "fullgrid=" g, $(NF-2), $(NF-1), $NF}'; done
