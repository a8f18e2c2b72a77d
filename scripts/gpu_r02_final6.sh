# round-2 final evidence (after the pack multiply change): GPU tests, smoke, bench lines of
# configs 1-4, reference arm, torchrun N = 1, launch list
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 2400 python -m pytest tests/ -x -v -m gpu --timeout 900 > gpurun_out/pytest_final6.log 2>&1; tail -3 gpurun_out/pytest_final6.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/f6_c1.json 2> gpurun_out/f6_c1.err; echo c1=$?
timeout 900 python bench.py --config 3 --steps 20 --warmup 5 > gpurun_out/f6_c3.json 2> gpurun_out/f6_c3.err; echo c3=$?
for c in 2 4; do
  timeout 1500 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/f6_c$c.json 2> gpurun_out/f6_c$c.err; echo c$c=$?
done
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/f6_ref.json 2> gpurun_out/f6_ref.err; echo ref=$?
for c in 1 2; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 2991$c \
    bench.py --gpus 1 --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/f6_tr$c.json 2> gpurun_out/f6_tr$c.err; echo tr$c=$?
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/f6_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/f6_ncu_launch.log 2>&1; echo ncu=$?
