python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CF_TEST_KNOBS="2=1" timeout 1800 python -m pytest tests -m gpu -x -v 2>&1 | grep -E "PASSED|FAILED|Error|info" | tail -8
