# the whole GPU suite plus the hull bench at 1e8 and the hull launch list
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python scripts/hull_bench.py --sizes 1e8 --out gpurun_out/hull_bench.txt > gpurun_out/hull_bench.log 2>&1; echo bench_rc=$?
cat gpurun_out/hull_bench.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/hull_launches.csv python scripts/hull_prof.py > gpurun_out/hull_prof.log 2>&1; echo ncu_rc=$?
python scripts/launch_summary.py gpurun_out/hull_launches.csv > gpurun_out/hull_launches.txt; cat gpurun_out/hull_launches.txt
