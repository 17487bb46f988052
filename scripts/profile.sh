# ncu evidence for the bench workload (1 GPU).  Outputs in gpurun_out/.
set -x
B="python bench.py --no-e2e --no-cpu-baseline"
# 1) launch list of our kernels (cold-cache, serialised: compare shares)
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
   -k regex:"k1_|k2_|k3_|k4_|k_gather" -c 12 --csv --log-file gpurun_out/launches_normal_1e9.csv \
   $B --steps 4 --warmup 2 > gpurun_out/ncu_launch_bench.log 2>&1; echo "launch rc=$?"
# 2) full capture of the two hot kernels
for K in k2_filter k1_extremes; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
     -o gpurun_out/prof_${K}_normal_1e9 $B --steps 2 --warmup 1 > gpurun_out/ncu_full_${K}.log 2>&1; echo "full $K rc=$?"
done
# 3) the other configs at 1e8 and the 1e4 latency case
for D in normal circle displaced; do
  timeout 300 $B --dist $D --n 1e8 --steps 50 --warmup 5 > gpurun_out/bench_${D}_1e8.json 2>&1; echo "bench $D rc=$?"
done
timeout 300 $B --dist normal --n 1e4 --steps 200 --warmup 10 > gpurun_out/bench_normal_1e4.json 2>&1
timeout 300 $B --dist circle --n 1e9 --steps 20 --warmup 3 > gpurun_out/bench_circle_1e9.json 2>&1
timeout 300 $B --dist displaced --n 1e9 --steps 20 --warmup 3 > gpurun_out/bench_displaced_1e9.json 2>&1
tail -n 2 gpurun_out/bench_*.json
