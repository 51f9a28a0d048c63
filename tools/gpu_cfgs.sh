# usage: bash tools/gpu_cfgs.sh TAG -- bench line per config + c5 with the jet developed + heavy A/B
TAG=${1:-r01e}
mkdir -p gpurun_out
timeout 1500 python tools/configs_bench.py $TAG > gpurun_out/cfgs_$TAG.log 2>&1; echo cfgs_rc=$?
timeout 600 python bench.py --config c5 --steps 20 --warmup 500 --no-cpu --no-e2e > gpurun_out/c5w500_$TAG.log 2>&1; echo c5_rc=$?
for w in 400 1000; do
  timeout 300 python tools/heavy_ab.py $w 10 > gpurun_out/hab_${w}_$TAG.log 2>&1
  DSMC_STATIC_CELLS=1 timeout 300 python tools/heavy_ab.py $w 10 > gpurun_out/hab_${w}_static_$TAG.log 2>&1
done
tail -n1 gpurun_out/hab_*_$TAG.log
