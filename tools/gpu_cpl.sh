mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_cpl.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu_cpl.log
for C in 1 2; do
  DSMC_CPL=$C timeout 300 python bench.py --n-runs 16 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/cpl$C.log 2>&1
  DSMC_CPL=$C timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/cpl${C}_256.log 2>&1
  echo CPL=$C; python tools/summ_bench.py gpurun_out/cpl$C.log gpurun_out/cpl${C}_256.log | grep -E "ms/step|collide"
done
