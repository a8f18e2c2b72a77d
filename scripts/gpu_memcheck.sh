# compute-sanitizer memcheck (one tool) over one case of every kernel path + a small plan
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python -m pytest tests/test_gpu.py -q -x -k "test_pair_small_path and 3-0 or test_pair_tensor_core_path and 8 or test_pair_complex128_dmma_path and 1 or test_pair_skinny_path and 2-0 or test_pair_wide_path and 1-0 or test_config0_complex128" > gpurun_out/mc_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 --log-file gpurun_out/memcheck.log python -m pytest tests/test_gpu.py -q -x -k "test_pair_small_path and 3-0 or test_pair_tensor_core_path and 8 or test_pair_complex128_dmma_path and 1 or test_pair_skinny_path and 2-0 or test_pair_wide_path and 1-0 or test_config0_complex128" > gpurun_out/mc_run.log 2>&1
echo memcheck_rc=$?
tail -3 gpurun_out/mc_plain.log gpurun_out/mc_run.log; tail -5 gpurun_out/memcheck.log
