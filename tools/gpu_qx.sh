timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k quantile_extremes 2>&1 | tail -3 > gpurun_out/pytest_qx.txt
