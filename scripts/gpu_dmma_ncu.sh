# ncu --set full (with source) of configs[3]'s dominant gathered DMMA launch (7th DMMA launch)
python -c "import __graft_entry__ as g; g.build()" || exit 1
ncu --set full --clock-control none --import-source on -k regex:zgemm_dmma_gather --launch-skip 6 -c 1 -o gpurun_out/dmma_dom -f python scripts/prof_dump.py 3 0 100 > gpurun_out/dmma_ncu.log 2>&1
echo ncu=$?
ncu -i gpurun_out/dmma_dom.ncu-rep --page source --csv --print-source sass > gpurun_out/dmma_dom_source.csv 2>&1
ncu -i gpurun_out/dmma_dom.ncu-rep --page raw --csv > gpurun_out/dmma_dom_raw.csv 2>&1
ncu -i gpurun_out/dmma_dom.ncu-rep --page details --csv > gpurun_out/dmma_dom_details.csv 2>&1
ls -la gpurun_out/dmma_dom*
