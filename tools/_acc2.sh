bash tools/gpu_variants.sh acc2 "f4 acc2"
DSMC_LIB=_ab/lib_acc2.so timeout 600 python tools/c5_timed.py 300 20 > gpurun_out/c5a_acc2.log 2>&1; tail -1 gpurun_out/c5a_acc2.log | cut -c1-200
DSMC_LIB=_ab/lib_acc2.so timeout 900 python -m pytest -x -q -m gpu -p no:cacheprovider tests > gpurun_out/pytest_acc2.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_acc2.log
