# parity of the in-tree build, then a same-box A/B against ab_alt/ (1 GPU)
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_robustness.py -q -x > gpurun_out/pytest_parity.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_parity.log
SIZES="${SIZES:-1e8 1e9}" bash scripts/ab_lib.sh > gpurun_out/ab.txt 2>&1
cat gpurun_out/ab.txt
