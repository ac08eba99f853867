bash tools/ab.sh "paper_2507_10150_b200/libpfsched.so tools/variants/nc3.so tools/variants/nc6m8.so tools/variants/nc3m10.so" "5" > gpurun_out/ab23.txt 2>&1
