mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_split.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu_split.log
for SP in 0 1; do
DSMC_SPLIT=$SP timeout 300 python bench.py --n-runs 16 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/split$SP.log 2>&1
DSMC_SPLIT=$SP timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/split${SP}_256.log 2>&1
echo SPLIT=$SP; python tools/summ_bench.py gpurun_out/split$SP.log gpurun_out/split${SP}_256.log | grep -E "ms/step|collide|stage|ntc"
done
