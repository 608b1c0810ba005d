T=r02m; O=gpurun_out/$T; mkdir -p $O
export EXTRA_FILES="tests/test_gpu_pnp.py tests/test_gpu_decode.py tests/test_gpu_fusion_engines.py"
export SUBSET="match_many_small_pairs or match_tiny_pairs or match_golden_cases or voxel_fusion_vs_oracle or voxel_partials or registration_edges_vs_golden or register_chain_global_poses or homography_ransac_golden_batched or retrieval_golden or local_candidates_golden or kernels_nn_query_golden or pnp_golden or noise_free or binned_fusion_vs_oracle or binned_points"
bash tools/sanitize.sh $T
