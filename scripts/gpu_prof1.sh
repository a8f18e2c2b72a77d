set -x
python scripts/prof_gemm.py 13 13 12 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:cgemm -s 2 -c 1 -o gpurun_out/prof_cgemm python scripts/prof_gemm.py 13 13 12 > gpurun_out/ncu_cgemm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pack -s 4 -c 1 -o gpurun_out/prof_pack python scripts/prof_gemm.py 13 13 12 > gpurun_out/ncu_pack.log 2>&1
python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
cat gpurun_out/prof_plain.log; tail -3 gpurun_out/ncu_cgemm.log gpurun_out/ncu_pack.log gpurun_out/ncu_launch.log
