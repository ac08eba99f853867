set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo pytest=$?
timeout 300 python bench.py > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:admit_kernel -c 1 -o gpurun_out/prof_r1b python tools/prof_admit.py --config 5 --ticks 2 > gpurun_out/ncu1.log 2>&1; echo ncu=$?
