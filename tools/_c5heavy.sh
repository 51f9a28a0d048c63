timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_collide_heavy" -s 1000 -c 2 -o gpurun_out/prof_c5heavy python tools/prof_step.py c5 4 500 2 > gpurun_out/ncu_c5heavy.log 2>&1; echo rc=$?
bash tools/ncu_export.sh gpurun_out/prof_c5heavy.ncu-rep "k_collide_heavy"
