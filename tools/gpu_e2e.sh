for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_e2e$i.json 2> gpurun_out/bench_e2e.err; done
timeout 300 python bench.py --config 4 --no-cpu-baseline > gpurun_out/bench_e2e_c4.json 2>> gpurun_out/bench_e2e.err
