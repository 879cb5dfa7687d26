# Final validation + profile round on one GPU box: tests, smoke, bench, reference arm, launch list, ncu full
#   gpurun -- bash tools/gpu_final_round.sh   (edit the tag below per round)
mkdir -p gpurun_out
bash tools/gpu_validate.sh
bash tools/gpu_profile_round.sh r2r
