# Round-2 final record after the device-hull work: GPU suite, smoke, the
# default bench line (with the a8 hull object), the hull bench with the host
# comparison, the device-hull launch lists (1 GPU).
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -3 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench_rc=$?
timeout 900 python scripts/hull_bench.py --sizes 1e8 --out gpurun_out/hull_final.txt > gpurun_out/hull_final.log 2>&1; echo hull_rc=$?
cat gpurun_out/hull_final.txt
bash scripts/gpu_hull_sync_prof.sh
