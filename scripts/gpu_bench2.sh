set -x
timeout 1500 python bench.py > gpurun_out/bench_r01b.json 2> gpurun_out/bench_r01b.err; echo rc=$?
cat gpurun_out/bench_r01b.json
python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches2.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch2.log 2>&1
echo ncu_rc=$?
