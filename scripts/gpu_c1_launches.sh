# configs[1] bench plan: per-launch device times of one slice (pack shapes), raster group
# sweep (DRAM bytes, time, clock) of the dominant GEMM incl. non-power-of-two groups
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python scripts/prof_dump.py 1 32 0.0 > gpurun_out/dump1.log 2>&1; echo dump=$?
python scripts/dump_summary.py gpurun_out/dump1.log 40 > gpurun_out/dump1_summary.txt
NO_FULL=1 GROUPS_M="3 4 5 6" timeout 1200 bash scripts/gpu_gemm_traffic.sh > gpurun_out/gsweep.log 2>&1
grep "G=" gpurun_out/gsweep.log
