# Round-2 GPU check: build, the GPU test suite, smoke, and the bench paths.
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout 1800 python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
for ex in nccl peer torch; do
  timeout 300 python bench.py --exchange $ex --points 1e8 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_w1_$ex.json 2> gpurun_out/bench_w1_$ex.err; echo bench_w1_${ex}_rc=$?
  tail -2 gpurun_out/bench_w1_$ex.err
done
for ex in torch peer; do
  CH_BENCH_SHARE_GPU=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --exchange $ex --points 1e8 --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_share_$ex.json 2> gpurun_out/bench_share_$ex.err; echo bench_share_${ex}_rc=$?
  tail -2 gpurun_out/bench_share_$ex.err
done
cat gpurun_out/bench_w1_*.json gpurun_out/bench_share_*.json | cut -c1-600
