mkdir -p gpurun_out
for cfg in c2 c3; do
for cw in 256 512 1024 0; do
if [ $cw = 0 ]; then unset DSMC_CAPW; else export DSMC_CAPW=$cw; fi
timeout 600 python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/${cfg}_capw$cw.log 2>&1; echo $cfg capw=$cw rc=$?; python tools/summ_bench.py gpurun_out/${cfg}_capw$cw.log | grep -E "ms/step|k_collide"
done
unset DSMC_CAPW
timeout 600 python bench.py --config $cfg --steps 20 --warmup 200 --no-cpu --no-e2e > gpurun_out/${cfg}_w200.log 2>&1; echo $cfg w200; python tools/summ_bench.py gpurun_out/${cfg}_w200.log | grep -E "ms/step|k_collide"
done
