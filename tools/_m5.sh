for v in mo0 mo1 mo3 mo4 mo14; do DSMC_LIB=_ab/lib_$v.so timeout 600 python tools/c5_timed.py 300 20 > gpurun_out/c5m_$v.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/c5m_$v.log').read().strip().split('\n')[-1]); k=d['kernels']
print('$v', round(d['ms_per_step_graph'],4), 'motion', k['k_motion']['ms'], k['k_motion']['GB/s'], 'collide', k['k_collide']['ms'], 'heavy', k.get('k_collide_heavy',{}).get('ms'))"; done
for v in mo0 mo4; do DSMC_LIB=_ab/lib_$v.so timeout 600 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/c3m_$v.log 2>&1; python tools/summ_bench.py gpurun_out/c3m_$v.log | head -3; done
