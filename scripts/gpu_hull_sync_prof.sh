set -x
mkdir -p gpurun_out
for d in displaced circle; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/hull_sync_$d.csv python scripts/hull_prof_sync.py $d > /dev/null 2>&1; echo ncu_rc=$?
python scripts/launch_summary.py gpurun_out/hull_sync_$d.csv > gpurun_out/hull_sync_$d.txt; cat gpurun_out/hull_sync_$d.txt
done
