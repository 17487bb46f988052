set -x
env | grep -i nccl
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout 600 python -m pytest tests/test_gpu_robustness.py -q > gpurun_out/pytest_rob.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_rob.log
timeout 300 python bench.py --exchange nccl --points 1e8 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_w1_nccl.json 2> gpurun_out/bench_w1_nccl.err; echo rc=$?
for ex in torch peer; do
  CH_BENCH_SHARE_GPU=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --exchange $ex --points 1e8 --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_share_$ex.json 2> gpurun_out/bench_share_$ex.err; echo bench_share_${ex}_rc=$?
  tail -3 gpurun_out/bench_share_$ex.err
done
CH_BENCH_SHARE_GPU=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29556 bench.py --gpus 2 --points 1e8 --steps 10 --warmup 3 > gpurun_out/bench_share_auto.json 2> gpurun_out/bench_share_auto.err; echo bench_share_auto_rc=$?
tail -3 gpurun_out/bench_share_auto.err
wc -l gpurun_out/bench_*.json
cat gpurun_out/bench_w1_nccl.json gpurun_out/bench_share_*.json | cut -c1-300
