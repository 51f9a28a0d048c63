# ncu --set full capture (with source) of the heavy-tile kernels on CONFIG after WARM steps
TAG=${1:-heavyc2}; CFG=${2:-c2}; WARM=${3:-3}; NR=${4:-64}
mkdir -p gpurun_out
SK=$((2 * WARM + 2))
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:k_collide_heavy -s $SK -c 2 -o gpurun_out/prof_$TAG python tools/prof_step.py $CFG $NR $WARM 2 > gpurun_out/ncu_$TAG.log 2>&1
echo ncu_rc=$?
tail -3 gpurun_out/ncu_$TAG.log
