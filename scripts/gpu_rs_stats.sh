set -x
mkdir -p gpurun_out
CH_NVCC_EXTRA="-DCH_RS_STATS" python -m paper_2303_10581_b200.build --force > gpurun_out/build_stats.log 2>&1; echo build_rc=$?
timeout 300 python scripts/hull_prof.py > gpurun_out/rs_stats.log 2>&1; echo rc=$?
grep rs_stats gpurun_out/rs_stats.log | head -20
