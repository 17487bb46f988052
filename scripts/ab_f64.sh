# A/B of a compile-time K2 variant on f64 storage: default build vs CH_NVCC_EXTRA="$AB" (1 GPU)
B="python bench.py --no-e2e --no-cpu-baseline --steps ${STEPS:-30} --warmup 3"
for V in base alt; do
  if [ $V = alt ]; then CH_NVCC_EXTRA="$AB" python -c "import paper_2303_10581_b200.build as b; b.build(force=True)"; fi
  for N in ${SIZES:-1e9 1e8}; do for D in ${DISTS:-normal circle displaced}; do
    timeout 300 $B --storage ${S:-f64} --dist $D --points $N 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print(f\"$V {d['config']['workload']:28s} {d['value']:8.2f} Gpts/s k1 {r['k1_ms']:.3f} k2 {r['k2_ms']:.3f} ({r['k2_gbs']:.0f} GB/s) clk {d['clocks']['sm_mhz']} {d['clocks']['reasons']}\")"
  done; done
done
