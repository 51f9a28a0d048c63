bash tools/gpu_c5prof.sh r02e 500
bash tools/ncu_export.sh gpurun_out/prof_c5_r02e.ncu-rep "k_collide<|k_motion<"
bash tools/gpu_round.sh r02e
bash tools/ncu_export.sh gpurun_out/prof_full_r02e.ncu-rep "k_collide<"
du -sh gpurun_out
