# usage: bash tools/gpu_check2.sh TAG -- all GPU tests, the default bench line, c5 after 300 steps
TAG=${1:-chk}
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -m gpu -p no:cacheprovider tests > gpurun_out/pytest_$TAG.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pytest_$TAG.log
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/bench_$TAG.log 2>&1; echo bench_rc=$?; python tools/summ_bench.py gpurun_out/bench_$TAG.log  2>/dev/null | head -8 || true
timeout 600 python tools/c5_timed.py 300 20 > gpurun_out/c5_$TAG.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/c5_$TAG.log').read().strip().split('\n')[-1]); k=d['kernels']
print('c5', round(d['ms_per_step_graph'],4), 'motion', k['k_motion']['ms'], 'collide', k['k_collide']['ms'], 'heavy', k.get('k_collide_heavy',{}).get('ms'), d['phases'])"
