mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_hsort.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_hsort.log
timeout 300 python tools/heavy_ab.py 400 10 > gpurun_out/hab_400.log 2>&1; tail -2 gpurun_out/hab_400.log
timeout 300 python tools/heavy_ab.py 1000 10 > gpurun_out/hab_1000.log 2>&1; tail -2 gpurun_out/hab_1000.log
timeout 600 python bench.py --config c5 --steps 20 --warmup 500 --no-cpu --no-e2e > gpurun_out/c5_hsort.log 2>&1; echo c5 rc=$?; python tools/summ_bench.py gpurun_out/c5_hsort.log | head -16
