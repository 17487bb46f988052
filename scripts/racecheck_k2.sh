# racecheck of K2 with several super-tiles per CTA (ring reuse) for the listed libraries (1 GPU)
cat > /tmp/rc.py <<'PY'
import sys; sys.path.insert(0, ".")
import numpy as np, torch, synth, paper_2303_10581_b200 as chf
for dist, n in (("displaced", 5_000_003),):
    xy = synth.points(dist, n, seed=2, device="cuda")
    ws = chf.Workspace(n)
    s = chf.filter(xy, ws)
    torch.cuda.synchronize()
print("rc workload ok")
PY
L=paper_2303_10581_b200/libchfilter.so
cp $L /tmp/keep.so
for NP in $LIBS; do
  cp ${NP#*=} $L; touch $L
  timeout 900 compute-sanitizer --tool racecheck python /tmp/rc.py > gpurun_out/rc_${NP%%=*}.log 2>&1
  echo "${NP%%=*}: $(grep -E 'RACECHECK SUMMARY' gpurun_out/rc_${NP%%=*}.log)"
  grep -E "Race reported between" gpurun_out/rc_${NP%%=*}.log | sed 's/(const T1.*)+/+/' | sort | uniq -c | head -8
done
cp /tmp/keep.so $L; touch $L
