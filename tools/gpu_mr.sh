timeout 600 python -m pytest tests/test_multirank.py -x -q 2>&1 | tail -15 > gpurun_out/pytest_mr.txt
