for v in hv5 mv1 mv3 mv2; do DSMC_LIB=_ab/lib_$v.so timeout 600 python tools/c5_timed.py 300 20 > gpurun_out/c5m_$v.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/c5m_$v.log').read().strip().split('\n')[-1]); k=d['kernels']
print('c5 $v', round(d['ms_per_step_graph'],4), 'motion', k['k_motion']['ms'])"
for c in c3 c2; do DSMC_LIB=_ab/lib_$v.so timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/${c}m_$v.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/${c}m_$v.log').read().strip().split('\n')[-1]); k=d['roofline']['kernels']
print('$c $v', round(d['ms_per_step'],4), 'motion', k['k_motion']['ms'])"; done; done
