timeout 900 python tools/sim_table1.py > gpurun_out/sim_table1.txt 2>&1
timeout 1500 python tools/sim_table1.py --slots 64 --req 1600 > gpurun_out/sim_table1_s64.txt 2>&1
