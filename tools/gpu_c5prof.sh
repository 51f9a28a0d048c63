# usage: bash tools/gpu_c5prof.sh TAG [WARM] -- c5 timed kernels after WARM steps, then one ncu --set full
# capture of k_motion / k_scatter / k_collide_triage / k_collide_list / k_collide_heavy of the step after WARM
TAG=$1; W=${2:-500}
mkdir -p gpurun_out
timeout 900 python tools/c5_timed.py $W 20 > gpurun_out/c5timed_$TAG.log 2>&1; echo timed_rc=$?; tail -1 gpurun_out/c5timed_$TAG.log | cut -c1-600
timeout 1800 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"k_motion<|k_scatter|k_collide" -s $((W*6)) -c 6 -o gpurun_out/prof_c5_$TAG \
  python tools/prof_step.py c5 4 $W 2 > gpurun_out/ncu_c5_$TAG.log 2>&1; echo ncu_rc=$?
tail -2 gpurun_out/ncu_c5_$TAG.log
