mkdir -p gpurun_out
for cfg in c5 c4; do
w=3; [ $cfg = c5 ] && w=500
for arm in old new; do
if [ $arm = old ]; then export DSMC_LIB=_ab/libdsmc_old.so; else unset DSMC_LIB; fi
timeout 600 python bench.py --config $cfg --steps 10 --warmup $w --no-cpu --no-e2e > gpurun_out/ab5_${cfg}_$arm.log 2>&1; echo $cfg $arm; python tools/summ_bench.py gpurun_out/ab5_${cfg}_$arm.log | grep -E "ms/step|k_collide "
done
done
