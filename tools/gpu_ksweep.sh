mkdir -p gpurun_out
for K in 1 2 4 8; do
  timeout 300 python bench.py --n-runs 64 --steps 16 --warmup 4 --timed-steps 8 --no-cpu --no-e2e --reorder-every $K > gpurun_out/k$K.log 2>&1
  echo "K=$K"; python tools/summ_bench.py gpurun_out/k$K.log
done
