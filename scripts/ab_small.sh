# Small-n latency A/B of two prebuilt libraries (in-tree vs ALT, 1 GPU): scripts/small_n.py, twice each
L=paper_2303_10581_b200/libchfilter.so
cp $L /tmp/new_small.so
for R in 1 2; do
  cp /tmp/new_small.so $L; touch $L; echo "== new"; python scripts/small_n.py --sizes 1e3 4e3 1e4 2e4 3e4 --dists normal circle displaced
  cp ${ALT:-ab_alt/libchfilter.so} $L; touch $L; echo "== alt"; python scripts/small_n.py --sizes 1e3 4e3 1e4 2e4 3e4 --dists normal circle displaced
done
cp /tmp/new_small.so $L; touch $L
