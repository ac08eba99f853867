timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/pytest_ab16.txt
bash tools/ab.sh "tools/variants/head.so paper_2507_10150_b200/libpfsched.so" "4 5 3" > gpurun_out/ab16.txt 2>&1
