PFSCHED_LIB=tools/variants/sn4.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2 > gpurun_out/pytest_ab22.txt
bash tools/ab.sh "paper_2507_10150_b200/libpfsched.so tools/variants/sn2.so tools/variants/sn4.so" "2" > gpurun_out/ab22.txt 2>&1
