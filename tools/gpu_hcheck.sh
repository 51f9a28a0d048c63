mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_hc.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_hc.log
timeout 600 python bench.py --config c5 --steps 20 --warmup 500 --no-cpu --no-e2e > gpurun_out/c5_hc.log 2>&1; echo c5 rc=$?; python tools/summ_bench.py gpurun_out/c5_hc.log | grep -E "ms/step|k_collide"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/c4_hc.log 2>&1; echo c4 rc=$?; python tools/summ_bench.py gpurun_out/c4_hc.log | grep -E "ms/step|k_collide"
