# compute-sanitizer on the hot kernels at small n (1 GPU)
set -x
cat > /tmp/san.py <<'PY'
import sys; sys.path.insert(0, ".")
import numpy as np, torch, oracle, synth, paper_2303_10581_b200 as chf
for dist, n in (("displaced", 300_001), ("circle", 70_000), ("normal", 200_003), ("displaced", 5), ("circle", 10_000), ("normal", 4_100), ("displaced", 30_000), ("normal", 1_000)):
    xy = synth.points(dist, n, seed=1, device="cuda")
    ws = chf.Workspace(n)
    s = chf.filter(xy, ws).cpu().numpy()
    want, _ = oracle.filter_compact(xy.cpu().numpy())
    assert np.array_equal(s, want), dist
    chf.octagon_filter(xy, ws)
    hull, surv, st = chf.hull_end_to_end(xy, ws)
# K2 with several super-tiles per CTA (buffer reuse without a block barrier,
# the adaptive box), float64 and float32 storage
for dist, n in (("displaced", 5_000_003), ("normal", 5_000_003), ("circle", 3_000_001)):
    for st_ in ("f64", "f32"):
        xy = synth.points(dist, n, seed=2, device="cuda")
        if st_ == "f32":
            xy = xy.float()
        ws = chf.Workspace(n)
        s = chf.filter(xy, ws).cpu().numpy()
        want, _ = oracle.filter_compact(xy.double().cpu().numpy())
        assert np.array_equal(s, want), (dist, st_)
print("sanitize workload ok")
PY
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python /tmp/san.py > gpurun_out/sanitize_$tool.log 2>&1; echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.log
done
