# round-2 evidence: ncu --set full of the gathered DMMA (configs[3]) and of the fp16x2 pack on
# the bench plan's dominant shape; launch list of the default bench (cold-cache, serialised)
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:zgemm_dmma_gather -c 10 -o gpurun_out/r02_zgemm_gather -f python scripts/run_config.py 3 1 > /dev/null 2>&1; echo zg=$?
$NCU -k regex:pack_f16 -c 1 -o gpurun_out/r02_pack_f16 -f python scripts/prof_gemm.py 16 16 12 > /dev/null 2>&1; echo pk=$?
python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r02_bench_plain.json 2> gpurun_out/r02_bench_plain.err; echo b=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r02_ncu_launch.log 2>&1; echo ncu=$?
