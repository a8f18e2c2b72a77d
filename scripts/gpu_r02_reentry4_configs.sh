# re-entry session 4: bench lines of configs 3, 2, 4 and the torchrun (NCCL, N = 1) default at HEAD
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
for c in 3 2 4; do
  timeout 1200 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_re4_c$c.json 2> gpurun_out/bench_re4_c$c.err; echo c$c=$?
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29541 \
  bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_re4_tr1.json 2> gpurun_out/bench_re4_tr1.err; echo tr1=$?
for f in gpurun_out/bench_re4_*.json; do head -c 330 $f; echo; done
