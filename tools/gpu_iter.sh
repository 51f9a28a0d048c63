# usage: bash tools/gpu_iter.sh TAG  -- gpu tests + bench (n=16 and default)
TAG=${1:-it}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python bench.py --n-runs 16 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench16_$TAG.log 2>&1; echo bench16_rc=$?
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench256_$TAG.log 2>&1; echo bench256_rc=$?
TAG=$TAG python tools/summ_bench.py gpurun_out/bench16_$TAG.log gpurun_out/bench256_$TAG.log
