#!/usr/bin/env bash
# compute-sanitizer passes over a reduced -m gpu subset (run under gpurun):
#   tools/sanitize.sh TAG
# racecheck (shared-memory hazards), synccheck (barrier misuse) and memcheck
# (out-of-bounds / misaligned global accesses) on the matcher's small-unit
# batches, fusion, registration and the homography RANSAC kernels.
set -u
TAG=${1:?tag}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
SUBSET=${SUBSET:-"match_many_small_pairs or match_tiny_pairs or match_golden_cases or voxel_fusion_vs_oracle or registration_edges_vs_golden or register_chain_global_poses or homography_ransac_golden_batched or retrieval_golden or local_candidates_golden or kernels_nn_query_golden"}
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
    timeout 1500 $CS --tool $tool --target-processes all --print-limit 50 --error-exitcode 17 \
        python -m pytest tests/test_gpu_parity.py ${EXTRA_FILES:-} -m gpu -x -q -p no:cacheprovider -k "$SUBSET" \
        > "$OUT/sanitizer_$tool.log" 2>&1
    echo "$tool rc=$?"
    tail -3 "$OUT/sanitizer_$tool.log"
done
