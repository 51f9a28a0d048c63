# usage: bash tools/gpu_src.sh TAG [CONFIG NRUNS KREGEX SKIP]  -- one ncu --set full capture with source of one kernel
TAG=${1:-src}; CFG=${2:-c4}; NR=${3:-16}; KR=${4:-k_collide}; SK=${5:-3}
mkdir -p gpurun_out
python tools/prof_step.py $CFG $NR 3 2 > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$KR" -s $SK -c ${6:-1} -o gpurun_out/prof_$TAG python tools/prof_step.py $CFG $NR 3 2 > gpurun_out/ncu_$TAG.log 2>&1
echo ncu_rc=$?
tail -3 gpurun_out/ncu_$TAG.log
