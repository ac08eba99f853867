# Round-1 final measurement: tests, smoke, bench lines, reference arm, launch list.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_final.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/smoke_final.txt 2>&1
timeout 400 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
for c in 2 3 4; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2>/dev/null; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
