# Same-box A/B of several prebuilt libraries: LIBS="name=path ..." (1 GPU).
# Each library is swapped into the package in turn and the bench matrix run.
B="python bench.py --no-e2e --no-cpu-baseline --steps ${STEPS:-30} --warmup 3"
L=paper_2303_10581_b200/libchfilter.so
cp $L /tmp/intree.so
run() {
  for S in ${STORAGES:-f64 f32}; do for N in ${SIZES:-1e9}; do for D in ${DISTS:-normal circle displaced}; do
    timeout 300 $B --storage $S --dist $D --points $N 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print(f\"$1 {d['config']['workload']:28s} {d['value']:8.2f} Gpts/s k1 {r['k1_ms']:.3f} k2 {r['k2_ms']:.3f} ({r['k2_gbs']:.0f} GB/s) clk {d['clocks']['sm_mhz']} {d['clocks']['reasons']}\")"
  done; done; done
}
for R in $(seq ${ROUNDS:-1}); do
  for NP in $LIBS; do
    cp ${NP#*=} $L; touch $L; run ${NP%%=*}
  done
done
cp /tmp/intree.so $L; touch $L
