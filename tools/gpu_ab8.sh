PFSCHED_LIB=tools/variants/m10.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2 > gpurun_out/pytest_ab8.txt
bash tools/ab.sh "paper_2507_10150_b200/libpfsched.so tools/variants/m9.so tools/variants/m10.so tools/variants/m9ls32.so" "5 3" > gpurun_out/ab8.txt 2>&1
