timeout 600 python tools/prof_step.py c5 4 500 8 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_collide" -s 1500 --csv --log-file gpurun_out/c5_collide_launches.csv python tools/prof_step.py c5 4 500 8 > gpurun_out/c5l.log 2>&1; echo rc=$?
python - <<'P'
import csv
rows=list(csv.reader(open("gpurun_out/c5_collide_launches.csv")))
h=next(i for i,r in enumerate(rows) if "Kernel Name" in r)
ki=rows[h].index("Kernel Name"); vi=rows[h].index("Metric Value")
for r in rows[h+1:]:
    if len(r)>vi: print(r[ki].split("(")[0][:40], r[vi])
P
timeout 900 ncu --set full --clock-control none -k regex:"k_collide_triage" -s 500 -c 1 -o gpurun_out/prof_triage python tools/prof_step.py c5 4 500 2 > gpurun_out/ncu_triage.log 2>&1; echo rc=$?
bash tools/ncu_export.sh gpurun_out/prof_triage.ncu-rep
