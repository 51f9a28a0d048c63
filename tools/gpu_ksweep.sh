# usage: bash tools/gpu_ksweep.sh -- c4 (n = 256) ms/step per reorder period K
for K in 1 2 3 4; do timeout 600 python bench.py --steps 12 --warmup 4 --no-cpu --no-e2e --reorder-every $K > gpurun_out/ks$K.log 2>&1; python tools/summ_bench.py gpurun_out/ks$K.log | head -1; done
