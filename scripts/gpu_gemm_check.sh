# build, the GPU tests of the tensor-core paths, GEMM device times of a short-K and a
# long-K step (ncu gpu__time_duration), smoke
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -3
bash scripts/time_pair_ncu.sh 18 16 8 cgemm2p
bash scripts/time_pair_ncu.sh 16 16 8 cgemm2p
bash scripts/time_pair_ncu.sh 18 12 12 cgemm2_f16
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
