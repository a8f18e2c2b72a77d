# configs[2] / [4] bench plans: step paths and per-launch device times of one slice
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python scripts/plan_summary.py 2 33 256 > gpurun_out/plan_c2.log 2>&1
TN_SEEDS=256 timeout 900 python scripts/prof_dump.py 2 33 1.0 > gpurun_out/dump2.log 2>&1; echo dump2=$?
python scripts/dump_summary.py gpurun_out/dump2.log 25 > gpurun_out/dump2_summary.txt
timeout 1200 python scripts/plan_summary.py 4 32 1024 > gpurun_out/plan_c4.log 2>&1
TN_SEEDS=1024 timeout 1200 python scripts/prof_dump.py 4 32 1.0 > gpurun_out/dump4.log 2>&1; echo dump4=$?
python scripts/dump_summary.py gpurun_out/dump4.log 25 > gpurun_out/dump4_summary.txt
