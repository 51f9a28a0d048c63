bash tools/gpu_variants.sh v2d "v2b m16 fullwb16"
bash tools/gpu_variants.sh v2dK1 "m16 fullwb16" --reorder-every 1
bash tools/gpu_variants.sh v2dK3 "fullwb16" --reorder-every 3
