# ncu full capture of K2 on the circle and displaced workloads (1e8), 1 GPU
set -x
B="python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 1 --points ${N:-1e8}"
for D in ${DISTS:-circle displaced}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KERN:-k2_filter} -s 2 -c 1 \
     -o gpurun_out/prof_${KERN:-k2_filter}_${D}_${N:-1e8} $B --dist $D > gpurun_out/ncu_${D}.log 2>&1; echo "full $D rc=$?"
done
