bash tools/gpu_variants.sh v2h "cur sw1024 sw2048 sw4096"
DSMC_LIB=_ab/lib_sw2048.so timeout 900 python -m pytest -x -q -m gpu -p no:cacheprovider tests/test_gpu_parity.py > gpurun_out/pytest_sw2048.log 2>&1; echo sw2048_pytest=$?; tail -1 gpurun_out/pytest_sw2048.log
