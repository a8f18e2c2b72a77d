# ncu of the fp16x2 pack of a K-slab (the (16, 12, 16) step: X = 2^32 entries in 4 K-slabs)
python -c "import __graft_entry__ as g; g.build()" || exit 1
ncu --set full --clock-control none --import-source on -k regex:pack_f16 -c 2 -o gpurun_out/pack_slab -f python scripts/prof_gemm.py 16 12 16 > gpurun_out/pack_slab_ncu.log 2>&1
echo ncu=$?
ncu -i gpurun_out/pack_slab.ncu-rep --page details --csv > gpurun_out/pack_slab_details.csv 2>&1
ncu -i gpurun_out/pack_slab.ncu-rep --page source --csv --print-source sass > gpurun_out/pack_slab_source.csv 2>&1
