# compute-sanitizer over small GPU parity cases (memcheck, racecheck, synccheck)
export PYTHONUNBUFFERED=1
SEL="tests/test_gpu_parity.py::test_multi_tick_parity tests/test_gpu_parity.py::test_edge_cases_empty_and_ragged tests/test_gpu_parity.py::test_empty_conditional_support"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --target-processes all python -m pytest -x -q $SEL -k "not 128" > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_rc.txt
done
