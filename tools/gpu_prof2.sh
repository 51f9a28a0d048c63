# usage: bash tools/gpu_prof2.sh TAG KREGEX SKIP COUNT [CFG NRUNS]
TAG=$1; KR=$2; SK=$3; CN=$4; CFG=${5:-c4}; NR=${6:-16}
mkdir -p gpurun_out
python tools/prof_step.py $CFG $NR 3 2 > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$KR" -s $SK -c $CN -o gpurun_out/prof_$TAG python tools/prof_step.py $CFG $NR 3 2 > gpurun_out/ncu_$TAG.log 2>&1
echo ncu_rc=$?
tail -2 gpurun_out/ncu_$TAG.log
