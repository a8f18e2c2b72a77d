# gathered skinny: one CTA per item (TN_WIDE_FULLGRID=1, default) vs 4 CTAs per SM grid-stride
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu.py -x -q -m gpu -k "skinny" 2>&1 | tail -1
for v in 1 0 1 0; do TN_WIDE_FULLGRID=$v timeout 300 python scripts/prof_dump.py 3 0 0.01 2>&1 | awk '/-- second run --/{f=1} f' | grep -E "skinny|wide nb=11" | sed "s/^/full=$v /"; done
