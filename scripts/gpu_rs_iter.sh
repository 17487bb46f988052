# one iteration on the device hull's sort: look-back stats (debug build), then
# the normal build's hull tests, hull bench and launch list
set -x
mkdir -p gpurun_out
CH_NVCC_EXTRA="-DCH_RS_STATS" python -m paper_2303_10581_b200.build --force > gpurun_out/build_stats.log 2>&1; echo build_rc=$?
timeout 300 python scripts/hull_prof.py > gpurun_out/rs_stats.log 2>&1; echo rc=$?
grep rs_stats gpurun_out/rs_stats.log | head -20
python -m paper_2303_10581_b200.build --force > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout 900 python -m pytest tests -q -x -m gpu -k "hull" > gpurun_out/pytest_hull.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_hull.log
timeout 600 python scripts/hull_bench.py --sizes 1e8 --host-max 0 --out gpurun_out/hull_bench.txt > gpurun_out/hull_bench.log 2>&1; echo bench_rc=$?
cat gpurun_out/hull_bench.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/hull_launches.csv python scripts/hull_prof.py > gpurun_out/hull_prof.log 2>&1; echo ncu_rc=$?
python scripts/launch_summary.py gpurun_out/hull_launches.csv
