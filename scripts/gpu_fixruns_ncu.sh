mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"k_fix_runs" -c 1 -f -o gpurun_out/fixruns python scripts/hull_prof.py > /dev/null 2>&1; echo ncu_rc=$?
