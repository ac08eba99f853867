timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/pytest_ovr.txt
bash tools/ab.sh "tools/variants/head.so paper_2507_10150_b200/libpfsched.so" "5" > gpurun_out/ab_ovr.txt 2>&1
timeout 600 python tools/next_bench.py > gpurun_out/next_rows_ovr.txt 2>&1
