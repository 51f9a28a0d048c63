bash tools/gpu_tests.sh mfast
timeout 900 python tools/c5_timed.py 500 20 > gpurun_out/c5timed_mfast.log 2>&1; tail -1 gpurun_out/c5timed_mfast.log | cut -c1-900
timeout 900 python tools/configs_bench.py mfast > gpurun_out/cfgs_mfast.log 2>&1; tail -8 gpurun_out/cfgs_mfast.log
