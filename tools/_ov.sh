bash tools/gpu_variants.sh ov "mv1 ov1"
for v in mv1 ov1; do DSMC_LIB=_ab/lib_$v.so timeout 600 python tools/c5_timed.py 300 20 > gpurun_out/c5o_$v.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/c5o_$v.log').read().strip().split('\n')[-1]); k=d['kernels']
print('c5 $v', round(d['ms_per_step_graph'],4), 'collide', k['k_collide']['ms'], 'heavy', k['k_collide_heavy']['ms'])"; done
DSMC_LIB=_ab/lib_ov1.so timeout 900 python -m pytest -x -q -m gpu -p no:cacheprovider tests > gpurun_out/pytest_ov1.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_ov1.log
