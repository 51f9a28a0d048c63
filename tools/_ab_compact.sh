bash tools/gpu_tests.sh compact
timeout 900 python tools/c5_timed.py 500 20 > gpurun_out/c5timed_compact.log 2>&1; tail -1 gpurun_out/c5timed_compact.log | cut -c1-1200
DSMC_COMPACT=0 timeout 900 python tools/c5_timed.py 500 20 > gpurun_out/c5timed_nocompact.log 2>&1; tail -1 gpurun_out/c5timed_nocompact.log | cut -c1-120
timeout 900 python tools/configs_bench.py compact > gpurun_out/cfgs_compact.log 2>&1; tail -8 gpurun_out/cfgs_compact.log
