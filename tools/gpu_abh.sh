mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
for cfg in c2 c3 c5; do
w=3; [ $cfg = c5 ] && w=500; [ $cfg = c3 ] && w=600
for arm in old new; do
if [ $arm = old ]; then export DSMC_LIB=_ab/libdsmc_old.so; else unset DSMC_LIB; fi
timeout 600 python bench.py --config $cfg --steps 20 --warmup $w --no-cpu --no-e2e > gpurun_out/abh_${cfg}_$arm.log 2>&1; echo $cfg $arm; python tools/summ_bench.py gpurun_out/abh_${cfg}_$arm.log | grep -E "ms/step|k_collide_heavy"
done
done
