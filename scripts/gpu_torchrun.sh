set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 2 --warmup 1 --config 2 --no-cpu-baseline > gpurun_out/tr_c2.json 2> gpurun_out/tr_c2.err; echo rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/tr_c1.json 2> gpurun_out/tr_c1.err; echo rc=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29535 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/tr_ref.json 2> gpurun_out/tr_ref.err; echo rc=$?
tail -2 gpurun_out/tr_c2.err gpurun_out/tr_c1.err
