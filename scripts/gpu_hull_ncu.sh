# ncu --set full of the device hull's sort kernels on the 1e8 circle
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu -k "hull" > gpurun_out/pytest_hull.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_hull.log
timeout 600 python scripts/hull_bench.py --sizes 1e8 --host-max 0 --out gpurun_out/hull_bench.txt > gpurun_out/hull_bench.log 2>&1; echo bench_rc=$?
cat gpurun_out/hull_bench.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/hull_launches.csv python scripts/hull_prof.py > gpurun_out/hull_prof.log 2>&1; echo ncu_rc=$?
python scripts/launch_summary.py gpurun_out/hull_launches.csv
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"k_rs_pass|k_keys_hist|k_fix_runs|k_points|k_gather_x" -c 6 -f -o gpurun_out/hull_sort_full python scripts/hull_prof.py > gpurun_out/hull_ncu_full.log 2>&1; echo ncu_full_rc=$?
