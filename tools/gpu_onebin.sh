timeout 600 python -m pytest tests/test_gpu_override_and_bins.py -x -q 2>&1 | tail -3 > gpurun_out/pytest_onebin.txt
