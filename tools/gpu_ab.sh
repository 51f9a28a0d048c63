mkdir -p gpurun_out
for i in 1 2; do
DSMC_LIB=_ab/libdsmc_old.so timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab_old$i.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab_new$i.log 2>&1
python tools/summ_bench.py gpurun_out/ab_old$i.log gpurun_out/ab_new$i.log | grep -E "ms/step|collide|scatter|motion"
done
