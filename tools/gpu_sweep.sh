# usage: bash tools/gpu_sweep.sh TAG "LIB1 LIB2 ..." "CPB1 CPB2 ..." [NRUNS]  -- collide time per (lib, region size)
TAG=${1:-sw}; LIBS=${2:-_ab/lib_r768.so}; CPBS=${3:-256}; NR=${4:-16}
mkdir -p gpurun_out
for L in $LIBS; do for C in $CPBS; do
  DSMC_LIB=$L DSMC_CPB=$C timeout 300 python bench.py --n-runs $NR --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/sw_${TAG}.log 2>&1
  echo "$L cpb=$C $(python tools/summ_bench.py gpurun_out/sw_${TAG}.log | grep -E 'ms/step|k_collide ' | tr '\n' ' ')"
done; done
