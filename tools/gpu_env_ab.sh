# usage: bash tools/gpu_env_ab.sh TAG CONFIG "ENV_A" "ENV_B" ... -- A/B of environment switches on one box (each arm
# twice, interleaved): bench line of CONFIG, ms/step and the Interaction kernels
TAG=$1; CFG=$2; shift 2
mkdir -p gpurun_out
for i in 1 2; do n=0; for A in "$@"; do n=$((n+1))
  env $A timeout 600 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/${TAG}_${CFG}_a${n}_$i.log 2>&1
  python - "$CFG [$A]" "gpurun_out/${TAG}_${CFG}_a${n}_$i.log" <<'P'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().split("\n")[-1]); k = d["roofline"]["kernels"]
    print(sys.argv[1], "ms/step %.3f" % d["ms_per_step"], " ".join("%s %.3f" % (n, v["ms"]) for n, v in k.items() if "collide" in n or n in ("k_motion", "k_scatter", "k_predraw")),
          "C+S 8TB/s frac", d["roofline"]["phases"]["collide+sample"]["frac_8TBs"])
except Exception as e:
    print(sys.argv[1], "error", e, open(sys.argv[2]).read()[-300:])
P
done; done
