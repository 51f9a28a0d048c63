mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
for cfg in c1 c2; do
for w in 3 200; do
timeout 600 python bench.py --config $cfg --steps 20 --warmup $w --no-cpu --no-e2e > gpurun_out/${cfg}_w$w.log 2>&1; echo $cfg w$w; python tools/summ_bench.py gpurun_out/${cfg}_w$w.log | grep -E "ms/step|k_collide"
DSMC_LIB=_ab/libdsmc_old.so timeout 600 python bench.py --config $cfg --steps 20 --warmup $w --no-cpu --no-e2e > gpurun_out/${cfg}_w${w}_old.log 2>&1; echo $cfg w$w old; python tools/summ_bench.py gpurun_out/${cfg}_w${w}_old.log | grep -E "ms/step|k_collide"
done
done
