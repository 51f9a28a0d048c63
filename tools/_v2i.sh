bash tools/gpu_variants.sh v2i "cur f4"
VARENV="DSMC_CAPW=448" bash tools/gpu_variants.sh v2i448 "f4"
VARENV="DSMC_CAPW=416" bash tools/gpu_variants.sh v2i416 "f4"
DSMC_LIB=_ab/lib_f4.so timeout 900 python -m pytest -x -q -m gpu -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_parity_r2.py > gpurun_out/pytest_f4.log 2>&1; echo f4_pytest=$?; tail -1 gpurun_out/pytest_f4.log
