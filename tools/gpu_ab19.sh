PFSCHED_LIB=tools/variants/g16.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2 > gpurun_out/pytest_ab19.txt
bash tools/ab.sh "paper_2507_10150_b200/libpfsched.so tools/variants/g8.so tools/variants/g16.so tools/variants/g64.so" "5 3" > gpurun_out/ab19.txt 2>&1
