bash tools/gpu_variants.sh nets "nets7 nets6 nets5 nets4"
for v in nets7 nets5 nets4; do DSMC_LIB=_ab/lib_$v.so timeout 600 python tools/c5_timed.py 300 20 > gpurun_out/c5n_$v.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/c5n_$v.log').read().strip().split('\n')[-1]); k=d['kernels']
print('c5 $v', round(d['ms_per_step_graph'],4), 'collide', k['k_collide']['ms'], 'heavy', k.get('k_collide_heavy',{}).get('ms'))"; done
