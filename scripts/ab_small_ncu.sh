# ncu device durations of the one-launch small-n step (K5 / K6): in-tree vs ALT library (1 GPU)
L=paper_2303_10581_b200/libchfilter.so
cp $L /tmp/new_k6.so
for V in new alt; do
  if [ $V = new ]; then cp /tmp/new_k6.so $L; else cp ${ALT:-ab_alt/libchfilter.so} $L; fi; touch $L
  for d in normal circle displaced; do for n in 2000 10000 30000; do
    ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k5_|k6_" python scripts/k6_prof.py $d $n 12 2>/dev/null \
      | python -c "
import csv,sys
v=[float(r[-1]) for r in csv.reader(sys.stdin) if len(r)>5 and r[-3]=='gpu__time_duration.sum']
v=v[2:]; v.sort()
print('$V $d $n', 'median_ns', v[len(v)//2] if v else None, 'min_ns', v[0] if v else None)"
  done; done
done
cp /tmp/new_k6.so $L; touch $L
