# configs[3]: per-launch device times of one amplitude (TN_PROFILE_DUMP), aggregated per kernel class and shape
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
TN_SEEDS=4 timeout 600 python scripts/prof_dump.py 3 0 0.0 > gpurun_out/c3_dump.out 2> gpurun_out/c3_dump.log; echo rc=$?
python scripts/dump_summary.py gpurun_out/c3_dump.log 40
