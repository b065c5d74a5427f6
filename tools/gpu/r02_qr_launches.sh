set -x
mkdir -p gpurun_out
for s in "2048 257" "8192 1024"; do
  set -- $s
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_qr_${1}x${2}_launches.csv \
      python tools/prof_qr.py $1 $2 1 > /dev/null 2>&1; echo rc=$?
done
