bash tools/ab.sh "tools/variants/head.so paper_2507_10150_b200/libpfsched.so" "5 3" > gpurun_out/ab20.txt 2>&1
