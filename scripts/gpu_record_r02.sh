# Round-2 record: full GPU suite + bench matrix, then the ncu evidence and the default bench line (1 GPU)
bash scripts/bench_matrix.sh > gpurun_out/matrix.txt 2>&1
bash scripts/profile.sh > gpurun_out/profile.txt 2>&1
tail -30 gpurun_out/matrix.txt
