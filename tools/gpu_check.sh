set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 300 python bench.py --n-runs 16 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench16.log 2>&1; echo bench16_rc=$?
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench256.log 2>&1; echo bench256_rc=$?
tail -n 5 gpurun_out/smoke.log gpurun_out/pytest_gpu.log gpurun_out/bench16.log gpurun_out/bench256.log
