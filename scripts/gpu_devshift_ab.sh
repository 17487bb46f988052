# ch_hull_gpu_async (second round decided on the device) with chunks sized for m >> HG_DEV_SHIFT
for s in 2 0 1 3 2; do
  CH_NVCC_EXTRA="-DHG_DEV_SHIFT=$s" python -m paper_2303_10581_b200.build --force > /dev/null 2>&1
  timeout 900 python scripts/hull_bench.py --sizes 1e8 --dists displaced circle --host-max 0 --out gpurun_out/hb_$s.txt > /dev/null 2>&1
  echo "shift $s"; tail -2 gpurun_out/hb_$s.txt
done
python -m paper_2303_10581_b200.build --force > /dev/null 2>&1
