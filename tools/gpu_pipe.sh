timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_pipe.txt
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_pipe$i.json 2> gpurun_out/bench_pipe.err; done
