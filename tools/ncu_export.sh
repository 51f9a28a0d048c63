# usage: bash tools/ncu_export.sh REP [SRC_KERNEL_REGEX] -- export an ncu report to gzipped CSV pages
# (raw metrics, details, and the source/SASS page of one kernel) and drop the .ncu-rep, so that
# gpurun_out/ stays under the 64 MiB copy-back limit
REP=$1; KR=$2; B=${REP%.ncu-rep}
ncu -i $REP --page raw --csv --kernel-name-base demangled > ${B}_raw.csv 2>/dev/null
ncu -i $REP --page details --csv --kernel-name-base demangled > ${B}_details.csv 2>/dev/null
if [ -n "$KR" ]; then
  ncu -i $REP --page source --csv --kernel-name-base demangled -k regex:"$KR" --print-source cuda,sass > ${B}_src.csv 2>/dev/null
fi
gzip -9f ${B}_*.csv
ls -la ${B}_*.csv.gz
rm -f $REP
