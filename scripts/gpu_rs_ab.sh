# A/B of radix-sort build variants (CH_NVCC_EXTRA per variant): device hull
# launch list on the 1e8 circle.  usage: bash scripts/gpu_rs_ab.sh "<flagsA>" "<flagsB>" ...
mkdir -p gpurun_out
i=0
for fl in "$@"; do
  CH_NVCC_EXTRA="$fl" python -m paper_2303_10581_b200.build --force > gpurun_out/build_ab$i.log 2>&1 || { echo "build $i failed"; tail gpurun_out/build_ab$i.log; }
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/ab_launches$i.csv python scripts/hull_prof.py > gpurun_out/ab_prof$i.log 2>&1
  echo "== variant $i: '$fl'"
  python scripts/launch_summary.py gpurun_out/ab_launches$i.csv | head -8
  i=$((i+1))
done
