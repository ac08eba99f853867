timeout 900 python -m pytest tests/test_gpu_baselines.py tests/test_gpu_sim.py -x -q 2>&1 | tail -2 > gpurun_out/pytest_base.txt
timeout 600 python tools/next_bench.py > gpurun_out/next_rows_base.txt 2>&1
