# tests + group-kernel A/B + profile in one gpurun call
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/j4_pytest.txt 2>&1; echo pytest=$?
tail -1 gpurun_out/j4_pytest.txt
bash tools/gpu.sh groupab
bash tools/gpu.sh profile j4
