# ncu --set full capture (with source) of the heavy-tile kernel at c5 after WARM steps of the jet
TAG=${1:-heavy}; WARM=${2:-500}; NR=${3:-4}
mkdir -p gpurun_out
timeout 600 python tools/prof_step.py c5 $NR $WARM 2 > gpurun_out/plain_$TAG.log 2>&1; echo plain_rc=$?
# two heavy launches (one per size tier) per step
SK=$((2 * WARM + 2))
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:k_collide_heavy -s $SK -c 2 -o gpurun_out/prof_$TAG python tools/prof_step.py c5 $NR $WARM 2 > gpurun_out/ncu_$TAG.log 2>&1
echo ncu_rc=$?
tail -3 gpurun_out/ncu_$TAG.log
