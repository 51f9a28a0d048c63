# usage: bash tools/gpu_capw.sh CONFIG WARM "CAPW1 CAPW2 ..."  -- bench line per warp staging capacity
# (DSMC_CAPW; 0 = the library's own rule), e.g. bash tools/gpu_capw.sh c5 500 "256 512 0"
CFG=${1:-c5}; W=${2:-3}; CWS=${3:-"256 512 1024 0"}
mkdir -p gpurun_out
for cw in $CWS; do
  if [ "$cw" = 0 ]; then unset DSMC_CAPW; else export DSMC_CAPW=$cw; fi
  timeout 600 python bench.py --config $CFG --steps 20 --warmup $W --no-cpu --no-e2e > gpurun_out/capw_${CFG}_w${W}_$cw.log 2>&1
  echo "$CFG warm=$W capw=$cw rc=$?"; python tools/summ_bench.py gpurun_out/capw_${CFG}_w${W}_$cw.log | grep -E "ms/step|k_collide"
done
