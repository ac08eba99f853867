bash tools/ab.sh "paper_2507_10150_b200/libpfsched.so tools/variants/tail.so" "5 4" > gpurun_out/ab12.txt 2>&1
