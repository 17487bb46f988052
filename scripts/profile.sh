# ncu evidence for the bench workload (1 GPU).  Outputs in gpurun_out/.
set -x
B="python bench.py --no-e2e --no-cpu-baseline"
W=${WORKLOAD:-normal}
N=${N:-1e9}
# 1) launch list of our kernels (cold-cache, serialised: compare shares)
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
   -k regex:"k1_|k2_|k3_|k4_|k_gather" -c 12 --csv --log-file gpurun_out/launches_${W}_${N}.csv \
   $B --dist $W --points $N --steps 4 --warmup 2 > gpurun_out/ncu_launch_bench.log 2>&1; echo "launch rc=$?"
# 2) full capture of the two hot kernels
for K in k2_filter k1_extremes; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
     -o gpurun_out/prof_${K}_${W}_${N} $B --dist $W --points $N --steps 2 --warmup 1 > gpurun_out/ncu_full_${K}.log 2>&1; echo "full $K rc=$?"
done
# 3) the bench line itself (not under ncu)
timeout 600 python bench.py --dist $W --points $N > gpurun_out/bench_${W}_${N}_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
cat gpurun_out/bench_${W}_${N}_full.json
