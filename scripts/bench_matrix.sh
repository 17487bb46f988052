# parity tests + bench over the workload matrix (1 GPU); outputs in gpurun_out/
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
B="python bench.py --no-e2e --no-cpu-baseline"
for S in ${STORAGES:-f64 f32}; do for N in 1e9 1e8; do for D in normal circle displaced; do
  timeout 300 $B --storage $S --dist $D --points $N --steps ${STEPS:-50} --warmup 3 > gpurun_out/bench_${D}_${N}_${S}.json 2>gpurun_out/bench_${D}_${N}_${S}.err; echo "bench $S $D $N rc=$?"
done; done; done
timeout 300 python bench.py --no-e2e --no-cpu-baseline --dist normal --points 1e4 --steps 500 --warmup 20 > gpurun_out/bench_normal_1e4_f64.json 2>/dev/null
python - <<'PY'
import json,glob
f = lambda v, fmt: format(v, fmt) if v is not None else "-"
for fn in sorted(glob.glob("gpurun_out/bench_*_f*.json")):
    try: d=json.loads(open(fn).read().strip().splitlines()[-1])
    except Exception as e: print(fn, "ERR", e); continue
    r=d["roofline"]
    print(f"{d['config']['workload']:28s} {d['value']:8.2f} Gpts/s  step {d['ms_per_step']*1e3:9.1f} us  k1 {r['k1_ms']:.3f} ({f(r['k1_gbs'],'.0f')} GB/s)  k2 {r['k2_ms']:.3f} ({f(r['k2_gbs'],'.0f')} GB/s)  frac {r['frac']:.3f} step {d['hbm_frac']:.3f}  surv {d['survivors']}  clk {d['clocks']['sm_mhz']} {d['clocks']['reasons']}")
PY
