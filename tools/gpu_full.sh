# usage: bash tools/gpu_full.sh TAG : default bench (+launch list of the same command), full ncu of top kernels
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_$TAG.txt
lscpu | head -20 > gpurun_out/cpu_$TAG.txt
python bench.py > gpurun_out/bench_full_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_full_$TAG.csv python bench.py --no-e2e --no-cpu > gpurun_out/ncu_list_$TAG.log 2>&1
echo bench_rc=$?
tail -c 2500 gpurun_out/bench_full_$TAG.log
python tools/prof_step.py c4 256 3 2 > gpurun_out/plain_full_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_collide|k_scatter|k_motion" -s 12 -c 3 -o gpurun_out/prof_full_$TAG python tools/prof_step.py c4 256 3 2 > gpurun_out/ncu_full_$TAG.log 2>&1
echo ncu_rc=$?
