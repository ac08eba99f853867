timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/pytest_ab21.txt
bash tools/ab.sh "tools/variants/head.so paper_2507_10150_b200/libpfsched.so" "5 4" > gpurun_out/ab21.txt 2>&1
