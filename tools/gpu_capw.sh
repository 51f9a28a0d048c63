mkdir -p gpurun_out
for cw in 256 512 768 1024 2048; do
DSMC_CAPW=$cw timeout 600 python bench.py --config c5 --steps 20 --warmup 500 --no-cpu --no-e2e > gpurun_out/c5_capw$cw.log 2>&1; echo capw=$cw rc=$?; python tools/summ_bench.py gpurun_out/c5_capw$cw.log | grep -E "ms/step|k_collide"
done
