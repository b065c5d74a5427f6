set -x
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:cqr \
  --log-file gpurun_out/cqr_launches.csv python tools/time_cholqr.py 2048x256 > gpurun_out/cqr_ncu.log 2>&1; echo rc=$?
python - <<'PY'
import csv, collections
rows = list(csv.DictReader(l for l in open("gpurun_out/cqr_launches.csv") if l.startswith('"')))
per = collections.defaultdict(list)
for r in rows:
    if r["Metric Name"] == "gpu__time_duration.sum":
        per[r["Kernel Name"].split("(")[0]].append(float(r["Metric Value"]))
for k, v in per.items():
    v = sorted(v); print(f"{k:40s} n={len(v):4d} median={v[len(v)//2]:10.1f} min={v[0]:10.1f}")
PY
