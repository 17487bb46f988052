# A/B of the small-n step (K5 / K6): in-tree build ("new") vs ab_alt/libchfilter.so ("alt"); 1 GPU.
L=paper_2303_10581_b200/libchfilter.so
cp $L /tmp/new.so
for R in 1 2; do
  for V in new alt; do
    if [ $V = new ]; then cp /tmp/new.so $L; else cp ${ALT:-ab_alt/libchfilter.so} $L; fi
    echo "== $V"
    timeout 300 python scripts/small_n.py --sizes ${SIZES:-1e3 4e3 5e3 1e4 2e4 3e4} --iters 500 2>&1 | tail -13
  done
done
cp /tmp/new.so $L
