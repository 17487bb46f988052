# ncu full captures of K2 (1e8) for the listed dists/storages; reports in gpurun_out/
set -x
DISTS="${DISTS:-displaced circle}" STORAGES="${STORAGES:-f64 f32}" TAG=${TAG:-_r02} bash scripts/profile_k2_matrix.sh
