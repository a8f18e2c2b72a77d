# ncu --set full of configs[3]'s gathered batched skinny launch ((10, 4, 4, 7), complex128)
python -c "import __graft_entry__ as g; g.build()" || exit 1
ncu --set full --clock-control none --import-source on -k regex:bskinny -c 1 -o gpurun_out/bskinny -f python scripts/prof_dump.py 3 0 100 > gpurun_out/bskinny_ncu.log 2>&1
echo ncu=$?
ncu -i gpurun_out/bskinny.ncu-rep --page source --csv --print-source sass > gpurun_out/bskinny_source.csv 2>&1
ncu -i gpurun_out/bskinny.ncu-rep --page details --csv > gpurun_out/bskinny_details.csv 2>&1
ncu -i gpurun_out/bskinny.ncu-rep --page raw --csv > gpurun_out/bskinny_raw.csv 2>&1
