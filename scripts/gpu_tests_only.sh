set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests/ -x -q -m gpu -rA 2>&1 | grep -E "PASS|FAIL|Error|error|assert|passed|failed" | tail -80
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
