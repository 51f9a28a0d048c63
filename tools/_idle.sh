bash tools/gpu_variants.sh idle "idle idle2"
for v in idle idle2; do DSMC_LIB=_ab/lib_$v.so timeout 600 python tools/c5_timed.py 300 20 > gpurun_out/c5i_$v.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/c5i_$v.log').read().strip().split('\n')[-1]); k=d['kernels']
print('c5 $v', round(d['ms_per_step_graph'],4), 'collide', k['k_collide']['ms'], 'heavy', k.get('k_collide_heavy',{}).get('ms'), d['phases'])"; done
DSMC_LIB=_ab/lib_idle2.so timeout 900 python -m pytest -x -q -m gpu -p no:cacheprovider tests > gpurun_out/pytest_idle.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_idle.log
