PFSCHED_LIB=tools/variants/bpt2.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2 > gpurun_out/pytest_ab7.txt
PFSCHED_LIB=tools/variants/bpt8.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2 >> gpurun_out/pytest_ab7.txt
bash tools/ab.sh "paper_2507_10150_b200/libpfsched.so tools/variants/bpt2.so tools/variants/bpt8.so tools/variants/m9.so tools/variants/ls8.so tools/variants/ls32.so" "5 3 4" > gpurun_out/ab7.txt 2>&1
