for cw in 256 320 384 448 512 640; do DSMC_CAPW=$cw timeout 600 python tools/c5_timed.py 300 20 > gpurun_out/c5cw_$cw.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/c5cw_$cw.log').read().strip().split('\n')[-1]); k=d['kernels']
print('capw $cw', round(d['ms_per_step_graph'],4), 'collide', k['k_collide']['ms'], 'heavy', k.get('k_collide_heavy',{}).get('ms'))"; done
