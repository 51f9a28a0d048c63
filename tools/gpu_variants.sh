# usage: bash tools/gpu_variants.sh TAG "LIB1 LIB2 ..." [bench args] -- c4 bench per _ab/lib_X.so (X=inline: in-tree), 2 rounds
TAG=$1; LIBS=$2; shift 2
mkdir -p gpurun_out
for i in 1 2; do
for L in $LIBS; do
  if [ "$L" = inline ]; then E=""; else E="DSMC_LIB=_ab/lib_$L.so"; fi
  env $E ${VARENV:-} timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e "$@" > gpurun_out/var_${TAG}_${L}_$i.log 2>&1
  python - gpurun_out/var_${TAG}_${L}_$i.log <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().split("\n")[-1]); k=d["roofline"]["kernels"]
    print("%-40s %.3f ms/step  collide %.3f  heavy %.3f  motion %.3f scatter %.3f  frac %.3f" % (sys.argv[1].split('/')[-1], d["ms_per_step"], k["k_collide"]["ms"], k.get("k_collide_heavy",{"ms":0})["ms"], k["k_motion"]["ms"], k["k_scatter"]["ms"], d["roofline"]["frac"]))
except Exception as e: print(sys.argv[1], "ERR", e, open(sys.argv[1]).read()[-300:])
PY
done
done
