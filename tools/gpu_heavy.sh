mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_heavy.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu_heavy.log
timeout 900 python bench.py --config c5 --steps 20 --warmup 300 --no-cpu --no-e2e --timed-steps 4 > gpurun_out/cfg_c5_w300_h.log 2>&1
echo "c5w300 rc=$?"; python tools/summ_bench.py gpurun_out/cfg_c5_w300_h.log | head -14
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench256_h.log 2>&1; python tools/summ_bench.py gpurun_out/bench256_h.log | grep -E "ms/step|collide"
