timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/pytest_ab10.txt
bash tools/ab.sh "paper_2507_10150_b200/libpfsched.so tools/variants/w32.so" "4" > gpurun_out/ab10.txt 2>&1
bash tools/ab.sh "paper_2507_10150_b200/libpfsched.so" "5 3 2" >> gpurun_out/ab10.txt 2>&1
