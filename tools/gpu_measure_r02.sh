# usage: bash tools/gpu_measure_r02.sh TAG -- GPU tests (with prints), c4 sweep, NEXT-1 A/B, all-config bench lines
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -m gpu -p no:cacheprovider -rA -s tests > gpurun_out/pytest_$TAG.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pytest_$TAG.log
grep -E "^full c2|^c1:|^c2_small:|^c3_small:|^c5_small:" gpurun_out/pytest_$TAG.log
timeout 1200 python tools/sweep_c4.py $TAG > gpurun_out/sweep_$TAG.log 2>&1; echo sweep_rc=$?
for w in 400 1000; do
  timeout 600 python tools/heavy_ab.py $w 20 > gpurun_out/hab_${w}_$TAG.log 2>&1
  DSMC_STATIC_CELLS=1 timeout 600 python tools/heavy_ab.py $w 20 > gpurun_out/hab_${w}_static_$TAG.log 2>&1
  tail -1 gpurun_out/hab_${w}_$TAG.log; tail -1 gpurun_out/hab_${w}_static_$TAG.log
done
timeout 1500 python tools/configs_bench.py $TAG > gpurun_out/cfgs_$TAG.log 2>&1; echo cfgs_rc=$?
