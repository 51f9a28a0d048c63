# usage: bash tools/gpu_round.sh TAG -- round artefacts: bench line, ncu launch list of the
# same command, ncu --set full of k_motion/k_scatter/k_collide (c4 n=256, one reorder and one
# non-reorder step: K = 2 alternates them)
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_$TAG.txt
lscpu | head -20 > gpurun_out/cpu_$TAG.txt
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/bench_$TAG.log | cut -c1-400
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --no-e2e --no-cpu > gpurun_out/ncu_list_$TAG.log 2>&1; echo list_rc=$?
timeout 900 python tools/prof_step.py c4 256 3 2 > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 1800 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"k_motion<|k_scatter|k_collide<" -s 9 -c 6 -o gpurun_out/prof_full_$TAG \
  python tools/prof_step.py c4 256 3 2 > gpurun_out/ncu_full_$TAG.log 2>&1
echo full_rc=$?
