# usage: bash tools/gpu_c5_env_ab.sh TAG WARM "ENV_A" "ENV_B" ... -- A/B of environment switches on c5 after WARM steps
# (tools/c5_timed.py; each arm twice, interleaved): graph ms/step and the Interaction kernels
TAG=$1; W=$2; shift 2
mkdir -p gpurun_out
for i in 1 2; do n=0; for A in "$@"; do n=$((n+1))
  env $A timeout 600 python tools/c5_timed.py $W 20 > gpurun_out/${TAG}_c5_a${n}_$i.log 2>&1
  python - "c5 [$A]" "gpurun_out/${TAG}_c5_a${n}_$i.log" <<'P'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().split("\n")[-1]); k = d["kernels"]
    print(sys.argv[1], "ms/step %.3f" % d["ms_per_step_graph"], " ".join("%s %.3f" % (n, v["ms"]) for n, v in k.items() if "collide" in n or n in ("k_motion", "k_scatter")))
except Exception as e:
    print(sys.argv[1], "error", e, open(sys.argv[2]).read()[-300:])
P
done; done
