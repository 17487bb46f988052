# bench lines with the separately timed hull object (a8)
mkdir -p gpurun_out
for d in displaced circle normal; do
  timeout 600 python bench.py --steps 20 --warmup 3 --points 1e8 --dist $d --no-cpu-baseline --no-e2e > gpurun_out/bench_hull_$d.json 2> gpurun_out/bench_hull_$d.err; echo "$d rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/bench_hull_$d.json').read().strip().splitlines()[-1]); print(d['config']['workload'], round(d['value'],1), d['hull'])"
done
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_hull_default.json 2> gpurun_out/bench_hull_default.err; echo "default rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/bench_hull_default.json').read().strip().splitlines()[-1]); print(d['config']['workload'], round(d['value'],1), d['hull'])"
