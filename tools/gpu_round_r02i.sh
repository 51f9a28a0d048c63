# usage: bash tools/gpu_round_r02i.sh -- round-2 closing artefacts (fourth session: float3 staging): c4 bench line,
# launch list and ncu --set full (gpu_round.sh), c5 after 500 steps with ncu, every config, the c4
# batching sweep, the NEXT-1 heavy-queue A/B, and the driver's contract invocations
T=r02i
bash tools/gpu_round.sh $T
bash tools/ncu_export.sh gpurun_out/prof_full_$T.ncu-rep "k_collide<"
bash tools/gpu_c5prof.sh $T 500
bash tools/ncu_export.sh gpurun_out/prof_c5_$T.ncu-rep "k_collide_list<|k_motion<"
timeout 900 python tools/configs_bench.py $T > gpurun_out/cfgs_$T.log 2>&1; tail -8 gpurun_out/cfgs_$T.log
timeout 900 python tools/sweep_c4.py $T > gpurun_out/sweep_$T.log 2>&1; tail -9 gpurun_out/sweep_$T.log
timeout 300 python tools/heavy_ab.py 400 10 > gpurun_out/hab_400_$T.log 2>&1
DSMC_STATIC_CELLS=1 timeout 300 python tools/heavy_ab.py 400 10 > gpurun_out/hab_400_static_$T.log 2>&1
tail -n1 gpurun_out/hab_*_$T.log
bash tools/gpu_contract.sh > gpurun_out/contract_$T.log 2>&1; cat gpurun_out/contract_$T.log
du -sh gpurun_out
