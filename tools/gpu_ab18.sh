PFSCHED_LIB=tools/variants/t1.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2 > gpurun_out/pytest_ab18.txt
bash tools/ab.sh "paper_2507_10150_b200/libpfsched.so tools/variants/t1.so tools/variants/t2.so tools/variants/t2b.so tools/variants/t8.so" "5 3" > gpurun_out/ab18.txt 2>&1
