# ncu full captures of K2 over (dist, storage) at 1e8, 1 GPU; reports in gpurun_out/
set -x
B="python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 1 --points ${N:-1e8}"
for S in ${STORAGES:-f64 f32}; do for D in ${DISTS:-displaced circle}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_filter -s 2 -c 1 \
     -o gpurun_out/prof_k2_${D}_${S}_${N:-1e8}${TAG:-} $B --dist $D --storage $S > gpurun_out/ncu_${D}_${S}.log 2>&1; echo "full $D $S rc=$?"
done; done
