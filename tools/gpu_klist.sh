# usage: bash tools/gpu_klist.sh TAG "LIB1 LIB2" [CONFIG NRUNS] -- per-launch k_collide durations (ncu, serialized) per lib
TAG=$1; LIBS=$2; CFG=${3:-c4}; NR=${4:-16}
for L in $LIBS; do
  DSMC_LIB=$L ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_collide" --csv python tools/prof_step.py $CFG $NR 0 12 2>/dev/null | grep k_collide | awk -F'","' '{print $NF}' | tr -d '"' | paste -sd' ' | sed "s|^|$L |"
done
