PFSCHED_LIB=tools/variants/pfn.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2 > gpurun_out/pytest_pfn.txt
bash tools/ab.sh "paper_2507_10150_b200/libpfsched.so tools/variants/pfn.so" "5 3 4" > gpurun_out/ab_pfn.txt 2>&1
