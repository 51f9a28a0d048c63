# usage: bash tools/gpu_prof.sh TAG CONFIG NRUNS   (tests, then ncu of the top kernels)
TAG=${1:-r1}; CFG=${2:-c4}; NR=${3:-16}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu_$TAG.log
python tools/prof_step.py $CFG $NR 3 1 > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python tools/prof_step.py $CFG $NR 3 1 > gpurun_out/ncu_list_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_collide|k_scatter|k_motion" -s 9 -c 3 -o gpurun_out/prof_$TAG python tools/prof_step.py $CFG $NR 3 1 > gpurun_out/ncu_$TAG.log 2>&1
echo ncu_rc=$?
tail -3 gpurun_out/ncu_$TAG.log
