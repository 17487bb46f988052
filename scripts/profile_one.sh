# usage: D=normal N=1e9 KERN=k2_filter TAG=x bash scripts/profile_one.sh
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KERN:-k2_filter} -s 2 -c 1 \
   -o gpurun_out/prof_${KERN:-k2_filter}_${D:-normal}_${N:-1e9}${TAG:-} python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 1 --points ${N:-1e9} --dist ${D:-normal} ${EXTRA:-} > gpurun_out/ncu_one.log 2>&1; echo "rc=$?"
