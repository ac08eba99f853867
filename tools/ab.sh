# A/B of libpfsched builds on one box: bench admit time per config (no CPU baseline).
# usage: bash tools/ab.sh "lib1 lib2 ..." "5 4 3"
LIBS=${1:-"paper_2507_10150_b200/libpfsched.so"}
CFGS=${2:-"5"}
for rep in 1 2; do
for c in $CFGS; do
  for L in $LIBS; do
    PFSCHED_LIB=$L timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 1 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$L cfg$c', 'admit_ms', round(d['config'].get('admit_kernel_ms',0),4), 'step_ms', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4))"
  done
done
done
