PFSCHED_LIB=tools/variants/mw8.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2 > gpurun_out/pytest_ab9.txt
bash tools/ab.sh "paper_2507_10150_b200/libpfsched.so tools/variants/mw4.so tools/variants/mw6.so tools/variants/mw8.so" "4" > gpurun_out/ab9.txt 2>&1
