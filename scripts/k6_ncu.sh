# ncu of the small-n one-launch step (K6 at 1e4, K5 at 2e3) on the current build; 1 GPU
set -x
mkdir -p gpurun_out/k6
for d in normal circle; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/k6_prof.py $d 10000 10 > gpurun_out/k6/dur_${d}_1e4.csv 2>&1
  ncu --set full --import-source on --clock-control none -k regex:k6 -s 3 -c 1 -o gpurun_out/k6/full_${d}_1e4 python scripts/k6_prof.py $d 10000 5 > /dev/null 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:k5 -s 3 -c 1 -o gpurun_out/k6/full_k5_normal_2e3 python scripts/k6_prof.py normal 2000 5 > /dev/null 2>&1
ls gpurun_out/k6
