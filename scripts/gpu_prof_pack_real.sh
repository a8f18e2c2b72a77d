# ncu --set full of pack launches inside the bench plan (configs[1], one slice, profiled path)
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
TN_PROFILE_DUMP=1000 python scripts/prof_dump.py 1 34 1000 > gpurun_out/pd_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pack_f16 -s 140 -c 3 -o gpurun_out/prof_pack_real -f python scripts/prof_dump.py 1 34 1000 > gpurun_out/ncu_pack_real.log 2>&1
echo ncu_rc=$?
