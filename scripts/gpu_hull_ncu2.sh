set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"k_chunk_chain|k_assemble_r|k_points" -c 3 -f -o gpurun_out/hull_chain_full python scripts/hull_prof.py > gpurun_out/hull_ncu2.log 2>&1; echo ncu_rc=$?
