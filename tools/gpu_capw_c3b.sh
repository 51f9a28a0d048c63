mkdir -p gpurun_out
for w in 3 600; do
for cw in 512 0; do
if [ $cw = 0 ]; then unset DSMC_CAPW; else export DSMC_CAPW=$cw; fi
timeout 600 python bench.py --config c3 --steps 20 --warmup $w --no-cpu --no-e2e > gpurun_out/c3b_w${w}_capw$cw.log 2>&1; echo c3 w$w capw=$cw; python tools/summ_bench.py gpurun_out/c3b_w${w}_capw$cw.log | grep -E "ms/step|k_collide"
done
done
