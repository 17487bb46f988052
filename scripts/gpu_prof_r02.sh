# Round-2 profiling: K2 displaced f64/f32 and K1 f32 full ncu captures (1e8, 1 GPU)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
DISTS=displaced STORAGES="f64 f32" TAG=_r02a bash scripts/profile_k2_matrix.sh
B="python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 1 --points 1e8"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_extremes -s 2 -c 1 \
   -o gpurun_out/prof_k1_normal_f32_r02a $B --dist normal --storage f32 > gpurun_out/ncu_k1.log 2>&1; echo k1 rc=$?
ls -la gpurun_out/
