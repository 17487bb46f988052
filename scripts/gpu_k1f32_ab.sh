# K1 float32 changes: the f32 K1 parity tests on the new build, then a same-box A/B of base / acc2 / new
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu -k "f32 or k1 or nonfinite or smoke" > gpurun_out/pytest_k1.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_k1.log
LIBS="base=ab_alt/base.so acc2=ab_alt/acc2.so new=ab_alt/new.so" STORAGES=f32 SIZES="1e9 1e8" ROUNDS=2 bash scripts/ab_libs.sh 2>&1 | grep -v "^+" > gpurun_out/ab_k1f32.txt
cat gpurun_out/ab_k1f32.txt
