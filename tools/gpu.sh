#!/usr/bin/env bash
# One parameterized driver for the GPU-box measurements (run under gpurun from the repo
# root; everything it writes goes to gpurun_out/, which gpurun copies back).
#
#   bash tools/gpu.sh tests            pytest -m gpu + smoke()
#   bash tools/gpu.sh bench [C...]      bench.py lines (default config 5, plus the given configs)
#   bash tools/gpu.sh reference         bench.py --impl reference (the CPU oracle arm)
#   bash tools/gpu.sh launches          ncu launch list (gpu__time_duration.sum) of a short bench run
#   bash tools/gpu.sh ncu C TAG         ncu --set full of the config-C admit kernel -> gpurun_out/TAG.ncu-rep
#   bash tools/gpu.sh ab "LIB..." "C..." A/B of libpfsched builds (PFSCHED_LIB) per config (tools/ab.sh)
#   bash tools/gpu.sh parity [ARGS]     tests/full_parity.py (full-size, every instance vs the oracle)
#   bash tools/gpu.sh ubench            tools/microbench/ubench (issue rates of the ops the kernel uses)
#   bash tools/gpu.sh sanitize          compute-sanitizer memcheck / racecheck / synccheck over GPU parity cases
#   bash tools/gpu.sh profile TAG [C]   ncu --set full of the 4th admit launch of config C (default 5) + raw / SASS csv
#                                       (read here with tools/ncu_keys.py, tools/sass_hist.py, tools/sass_blocks.py)
#   bash tools/gpu.sh final             tests, bench lines, oracle arm, launch list, ncu cfg 5/4, shard probe
#   bash tools/gpu.sh groupab           bench cfg 5 with admit_group_kernel (default) and with admit_kernel
#                                       (PFSCHED_GROUP_KERNEL=0) on one box
#
# Inputs: the in-tree libpfsched.so (built by __graft_entry__.build()), alternative builds
# for `ab` passed as paths (e.g. tools/variants/*.so from build.build(extra=[...], out=...)).
set -u
mode=${1:-tests}
shift || true
mkdir -p gpurun_out
case "$mode" in
  tests)
    timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest=$?"
    tail -2 gpurun_out/pytest_gpu.txt
    timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1; echo "smoke=$?" ;;
  bench)
    timeout 400 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench=$?"
    for c in "$@"; do
      timeout 300 python bench.py --config "$c" --no-cpu-baseline > "gpurun_out/bench_cfg$c.json" 2> "gpurun_out/bench_cfg$c.err"
      echo "cfg$c=$?"
    done ;;
  reference)
    timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
    echo "reference=$?" ;;
  launches)
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
      -k regex:"admit_kernel|admit_group_kernel|group_tables|update_hist|update_sorted|init_ring|hist_rows|sort_rows" \
      python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo "launches=$?" ;;
  ncu)
    c=${1:-5}; tag=${2:-admit_cfg$c}
    timeout 600 ncu --set full --import-source on --clock-control none -k regex:admit --launch-skip 3 -c 1 -o "gpurun_out/$tag" \
      python tools/prof_admit.py --config "$c" --ticks 4 > "gpurun_out/$tag.log" 2>&1; echo "ncu=$?" ;;
  ab)
    bash tools/ab.sh "$1" "${2:-5}" ;;
  parity)
    timeout 3000 python tests/full_parity.py "$@" > gpurun_out/full_parity.log 2>&1; echo "parity=$?"
    tail -12 gpurun_out/full_parity.log ;;
  ubench)
    ./tools/microbench/ubench > gpurun_out/ubench.txt 2>&1; echo "ubench=$?" ;;
  sanitize)
    sel='multi_tick or empty_conditional or two_live or (variant_parity and (tw2 or tw1_unpacked or big_lmax))'
    : > gpurun_out/sanitizer.txt
    for tool in memcheck racecheck synccheck; do
      echo "== compute-sanitizer --tool $tool (pytest -k \"$sel\"; one B200)" >> gpurun_out/sanitizer.txt
      timeout 1200 compute-sanitizer --tool $tool python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py \
        -q -x -k "$sel" >> gpurun_out/sanitizer.txt 2>&1
      echo "$tool=$?"
    done
    grep -E "SUMMARY|passed|failed" gpurun_out/sanitizer.txt ;;
  profile)
    tag=${1:-prof}; c=${2:-5}
    timeout 600 ncu --set full --import-source on --clock-control none -k regex:admit --launch-skip 3 -c 1 \
      -o "gpurun_out/$tag" python tools/prof_admit.py --config "$c" --ticks 4 > "gpurun_out/$tag.log" 2>&1; echo ncu=$?
    ncu -i "gpurun_out/$tag.ncu-rep" --page raw --csv > "gpurun_out/${tag}_raw.csv" 2>&1
    ncu -i "gpurun_out/$tag.ncu-rep" --page source --csv --print-source sass > "gpurun_out/${tag}_sass.csv" 2>&1 ;;
  groupab)
    for v in 1 0; do
      PFSCHED_GROUP_KERNEL=$v timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 --steps 100 --warmup 5 2>/dev/null \
        | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('group_kernel=$v', 'admit_ms', round(d['config']['admit_kernel_ms'], 4), 'step_ms', round(d['ms_per_step'], 4), d['config']['output_check'])"
    done ;;
  final)
    # the round-end evidence set: tests + smoke, bench lines cfg 5 (default) and 1-4, the oracle
    # arm, the launch list, ncu of the cfg 5 and cfg 4 admit kernels, the P-rank shard probe
    bash tools/gpu.sh tests
    bash tools/gpu.sh bench 1 2 3 4
    bash tools/gpu.sh reference
    bash tools/gpu.sh launches
    python tools/ncu_launches.py gpurun_out/launches_bench.csv "bench.py --steps 4 --warmup 3" > gpurun_out/launches_summary.txt 2>&1
    bash tools/gpu.sh profile final_cfg5 5
    bash tools/gpu.sh profile final_cfg4 4
    timeout 600 python tools/shard_probe.py > gpurun_out/shard_probe.txt 2>&1; echo "probe=$?" ;;
  *) echo "unknown mode $mode"; exit 2 ;;
esac
