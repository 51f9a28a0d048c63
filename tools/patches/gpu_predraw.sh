# usage: bash tools/gpu_predraw.sh TAG [CONFIGS] -- A/B of k_predraw (DSMC_PREDRAW=0/1) on one box: GPU tests with
# the default (on where eligible), then each config's bench line twice per arm, interleaved
TAG=${1:-pd}; CFGS=${2:-"c4 c3 c1"}
mkdir -p gpurun_out
timeout 1500 python -m pytest -x -q -m gpu -p no:cacheprovider tests > gpurun_out/pytest_$TAG.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_$TAG.log
for CFG in $CFGS; do for i in 1 2; do for A in 0 1; do
  DSMC_PREDRAW=$A timeout 600 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/${TAG}_${CFG}_pd${A}_$i.log 2>&1
  python - "$CFG pd=$A" "gpurun_out/${TAG}_${CFG}_pd${A}_$i.log" <<'P'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().split("\n")[-1]); k = d["roofline"]["kernels"]
    print(sys.argv[1], "ms/step %.3f" % d["ms_per_step"], " ".join("%s %.3f" % (n, v["ms"]) for n, v in k.items() if "collide" in n or n in ("k_motion", "k_scatter", "k_predraw")),
          "C+S 8TB/s frac", d["roofline"]["phases"]["collide+sample"]["frac_8TBs"])
except Exception as e:
    print(sys.argv[1], "error", e, open(sys.argv[2]).read()[-300:])
P
done; done; done
