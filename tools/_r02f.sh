bash tools/gpu_tests.sh r02f
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/b_c4.log 2>&1; tail -1 gpurun_out/b_c4.log | python tools/summ_bench.py /dev/stdin 2>/dev/null | head -5
python tools/summ_bench.py gpurun_out/b_c4.log gpurun_out/b_c4_compact.log | grep -E "ms/step|collide|triage"
