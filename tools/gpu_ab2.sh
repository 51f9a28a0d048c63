# usage: bash tools/gpu_ab2.sh TAG OLD_LIB [bench args...] -- GPU parity subset, then c4 bench A/B (old vs in-tree)
TAG=$1; OLD=$2; shift 2
mkdir -p gpurun_out
timeout 1500 python -m pytest -x -q -m gpu -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_parity_r2.py \
  > gpurun_out/pytest_$TAG.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_$TAG.log
for i in 1 2; do
DSMC_LIB=$OLD timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e "$@" > gpurun_out/ab_${TAG}_old$i.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e "$@" > gpurun_out/ab_${TAG}_new$i.log 2>&1
python tools/summ_bench.py gpurun_out/ab_${TAG}_old$i.log gpurun_out/ab_${TAG}_new$i.log | grep -E "ms/step|collide|scatter|motion"
done
