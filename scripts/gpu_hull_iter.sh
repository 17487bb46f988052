# device hull iteration: hull tests, hull bench (1e8), launch lists of ch_hull_gpu (displaced, circle)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu -k "hull" > gpurun_out/pytest_hull.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_hull.log
timeout 600 python scripts/hull_bench.py --sizes 1e8 --host-max 0 --out gpurun_out/hull_bench.txt > gpurun_out/hull_bench.log 2>&1; echo bench_rc=$?
cat gpurun_out/hull_bench.txt
bash scripts/gpu_hull_sync_prof.sh
