for v in hv1 hv4; do DSMC_LIB=_ab/lib_$v.so timeout 600 python tools/c5_timed.py 300 20 > gpurun_out/c5h_$v.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/c5h_$v.log').read().strip().split('\n')[-1]); k=d['kernels']
print('c5 $v', round(d['ms_per_step_graph'],4), 'collide', k['k_collide']['ms'], 'heavy', k.get('k_collide_heavy',{}).get('ms'))"; done
for v in hv1 hv4; do DSMC_LIB=_ab/lib_$v.so timeout 600 python bench.py --config c2 --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/c2h_$v.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/c2h_$v.log').read().strip().split('\n')[-1]); k=d['roofline']['kernels']
print('c2 $v', round(d['ms_per_step'],4), 'collide', k['k_collide']['ms'], 'heavy', k.get('k_collide_heavy',{}).get('ms'))"; done
DSMC_LIB=_ab/lib_hv4.so timeout 900 python -m pytest -x -q -m gpu -p no:cacheprovider tests > gpurun_out/pytest_hv1.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_hv1.log
