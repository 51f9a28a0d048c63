bash tools/gpu_src.sh r02nr c4 64 "k_collide<" 4 1
bash tools/gpu_src.sh r02re c4 64 "k_collide<" 3 1
