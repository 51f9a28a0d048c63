# usage: bash tools/gpu_sweep2.sh LIB "ENV1;ENV2;..." [NRUNS] -- collide time per env setting
L=$1; NR=${3:-16}
IFS=';' read -ra ENVS <<< "$2"
for E in "${ENVS[@]}"; do
  env $E DSMC_LIB=$L timeout 300 python bench.py --n-runs $NR --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/sw2.log 2>&1
  echo "$L [$E] $(python tools/summ_bench.py gpurun_out/sw2.log | grep -E 'ms/step|k_collide ' | tr '\n' ' ')"
done
