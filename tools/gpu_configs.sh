mkdir -p gpurun_out
for C in c1 c2 c3 c5; do
  timeout 600 python bench.py --config $C --steps 20 --warmup 3 --no-cpu --no-e2e --timed-steps 4 > gpurun_out/cfg_$C.log 2>&1
  echo "$C rc=$?"; python tools/summ_bench.py gpurun_out/cfg_$C.log | head -12
done
# c5 after the jet has developed (300 steps)
timeout 900 python bench.py --config c5 --steps 20 --warmup 300 --no-cpu --no-e2e --timed-steps 4 > gpurun_out/cfg_c5_w300.log 2>&1
echo "c5w300 rc=$?"; python tools/summ_bench.py gpurun_out/cfg_c5_w300.log | head -12
tail -3 gpurun_out/cfg_c5_w300.log | cut -c1-300
