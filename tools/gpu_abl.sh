# usage: bash tools/gpu_abl.sh CONFIG LIB... -- A/B of library builds in abl/ on one box: each twice,
# interleaved (c4 bench line, or c5 after 300 steps); prints ms/step and the collide kernels
CFG=$1; shift
mkdir -p gpurun_out
for i in 1 2; do for L in "$@"; do
  if [ "$CFG" = c4 ]; then
    DSMC_LIB=abl/lib_$L.so timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/abl_${L}_$i.log 2>&1
    python - "$L" "gpurun_out/abl_${L}_$i.log" <<'P'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().split("\n")[-1]); k = d["roofline"]["kernels"]
print(sys.argv[1], "ms/step %.3f" % d["ms_per_step"], " ".join("%s %.3f" % (n, v["ms"]) for n, v in k.items() if "collide" in n or n in ("k_motion", "k_scatter")))
P
  else
    DSMC_LIB=abl/lib_$L.so timeout 600 python tools/c5_timed.py 300 20 > gpurun_out/abl_${L}_$i.log 2>&1
    python - "$L" "gpurun_out/abl_${L}_$i.log" <<'P'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().split("\n")[-1]); k = d["kernels"]
print(sys.argv[1], "ms/step %.3f" % d["ms_per_step_graph"], " ".join("%s %.3f" % (n, v["ms"]) for n, v in k.items() if "collide" in n or n in ("k_motion", "k_scatter")))
P
  fi
done; done
