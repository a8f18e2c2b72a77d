# fp16x2 pack A/B on one box: the round-2 kernel (old) vs unrolled chunk-max shuffles and the
# exponent taken from the float's bits (new); libraries prebuilt in abtmp/ (not committed)
set -x
cp abtmp/lib_new.so paper_2208_01498_b200/libtn_b200.so
timeout 900 python -m pytest tests/test_gpu.py -x -q -m gpu -k "tensor_core or wide_dynamic or zero_chunk or error or k_slabs or in_bounds" 2>&1 | tail -2
for v in new old new old; do
  cp abtmp/lib_$v.so paper_2208_01498_b200/libtn_b200.so
  timeout 900 python bench.py --config 1 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/b1_$v.json 2> gpurun_out/b1_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/b1_$v.json'))
k=d['kernels']['pack_f16x2s_kernel']
print('$v', round(d['value']/1e12,1), d['clocks']['sm_mhz'], 'pack', round(k['ms'],1), round(k['share_of_step'],4), round(k['frac'],3), 'gemm', round(d['kernels']['cgemm2_f16x2s_kernel']['frac'],3))"
done
