set -x
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo rc=$?
cat gpurun_out/bench_default.json gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_default.err gpurun_out/bench_ref.err
