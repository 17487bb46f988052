set -x
mkdir -p gpurun_out
CUDA_LAUNCH_BLOCKING=1 timeout 600 python scripts/debug_hull_sort.py all 1e7 > gpurun_out/dbg_all.log 2>&1; echo rc=$?
cat gpurun_out/dbg_all.log | tail -30
timeout 600 compute-sanitizer --tool memcheck python scripts/debug_hull_sort.py cluster50k > gpurun_out/dbg_san.log 2>&1; echo rc=$?
grep -m 20 -A8 "Invalid\|ERROR\|error" gpurun_out/dbg_san.log | head -60
