# round-2 bench lines: default (with the oracle baseline), configs 2-4, the reference arm,
# and the torchrun (NCCL process group at N = 1) path of configs 1 and 2
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python bench.py > gpurun_out/bench_r02_c1.json 2> gpurun_out/bench_r02_c1.err; echo c1=$?
for c in 3 2 4; do
  timeout 1200 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_r02_c$c.json 2> gpurun_out/bench_r02_c$c.err; echo c$c=$?
done
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_r02_ref.json 2> gpurun_out/bench_r02_ref.err; echo ref=$?
for c in 1 2; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 2951$c \
    bench.py --gpus 1 --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r02_tr$c.json 2> gpurun_out/bench_r02_tr$c.err; echo tr$c=$?
done
