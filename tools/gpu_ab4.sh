bash tools/ab.sh "tools/variants/nocarve.so paper_2507_10150_b200/libpfsched.so" "5 3" > gpurun_out/ab4.txt 2>&1
timeout 300 ncu --section LaunchStats --section MemoryWorkloadAnalysis --section SpeedOfLight -k regex:admit_kernel -c 1 python tools/prof_admit.py --config 5 --ticks 1 > gpurun_out/ncu_ab4.txt 2>&1
