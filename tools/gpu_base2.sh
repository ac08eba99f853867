for L in paper_2507_10150_b200/libpfsched.so tools/variants/b8.so tools/variants/b2.so; do
  echo $L >> gpurun_out/next_rows_base2.txt
  PFSCHED_LIB=$L timeout 600 python tools/next_bench.py 2>&1 | head -2 >> gpurun_out/next_rows_base2.txt
done
