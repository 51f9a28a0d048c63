bash tools/gpu_round.sh r02g
bash tools/ncu_export.sh gpurun_out/prof_full_r02g.ncu-rep "k_collide<"
bash tools/gpu_c5prof.sh r02g 500
bash tools/ncu_export.sh gpurun_out/prof_c5_r02g.ncu-rep "k_collide_list<|k_motion<"
timeout 900 python tools/configs_bench.py r02g > gpurun_out/cfgs_r02g.log 2>&1; tail -8 gpurun_out/cfgs_r02g.log
du -sh gpurun_out
