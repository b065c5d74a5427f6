timeout 120 python tools/prof_build.py 6 2>&1 | tail -3
SKL_PROF_WARM_S=0.01 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file gpurun_out/build_launches.csv python tools/prof_build.py 3 > /dev/null 2>&1; echo ncu rc=$?
python - <<'PY'
import csv, collections
rows = list(csv.DictReader(l for l in open("gpurun_out/build_launches.csv") if l.startswith('"')))
per = collections.defaultdict(list)
for r in rows:
    if r["Metric Name"] == "gpu__time_duration.sum":
        per[r["Kernel Name"].split("(")[0][:60]].append(float(r["Metric Value"]))
for k, v in per.items():
    print(f"{k:60s} n={len(v):3d} mean={sum(v)/len(v)/1e3:8.1f}us")
PY
