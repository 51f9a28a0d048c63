# usage: bash tools/gpu_tests.sh TAG [pytest selectors...] -- GPU test run with a log under gpurun_out/
TAG=${1:-t}; shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > gpurun_out/gpu_$TAG.txt
# (the in-tree .so travels with the snapshot; build() is the driver's check)
timeout 3000 python -m pytest -x -q -m gpu -p no:cacheprovider "${@:-tests}" > gpurun_out/pytest_$TAG.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_$TAG.log
