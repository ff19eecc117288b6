timeout 900 python -m pytest tests/test_multigpu.py -x -q 2>&1 | tail -2
SKIP_TESTS=1 CTS=1.0 bash tools/n4_gd.sh
