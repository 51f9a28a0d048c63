for v in mo4 acc; do DSMC_LIB=_ab/lib_$v.so timeout 600 python tools/c5_timed.py 300 20 > gpurun_out/c5a_$v.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/c5a_$v.log').read().strip().split('\n')[-1]); k=d['kernels']
print('$v', round(d['ms_per_step_graph'],4), 'motion', k['k_motion']['ms'], 'collide', k['k_collide']['ms'], k['k_collide']['GB/s'], 'heavy', k.get('k_collide_heavy',{}).get('ms'), d['phases'])"; done
bash tools/gpu_variants.sh acc "mo4 acc"
