DSMC_LIB=abl/lib_9215b65.so timeout 600 python -m pytest -x -q -m gpu -p no:cacheprovider tests/test_gpu_parity.py -k heavy_tier_edge 2>&1 | tail -3
bash tools/gpu_tests.sh fix
python tools/_diag_det.py 550 0 1100
