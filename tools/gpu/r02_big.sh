timeout 600 python -m pytest tests/test_gpu_cholqr.py -q -x 2>&1 | tail -4
timeout 300 python tools/time_cholqr.py 2048x256 2048x600 8192x1024 2>&1 | tail -3
SKL_PROF_WARM_S=0.01 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file gpurun_out/big_launches.csv python tools/prof_qr.py 8192 1024 1 cholqr > /dev/null 2>&1; echo ncu rc=$?
python - <<'PY'
import csv, collections
rows = list(csv.DictReader(l for l in open("gpurun_out/big_launches.csv") if l.startswith('"')))
per = collections.defaultdict(list)
for r in rows:
    if r["Metric Name"] == "gpu__time_duration.sum":
        per[r["Kernel Name"].split("(")[0]].append(float(r["Metric Value"]))
for k, v in per.items():
    print(f"{k:40s} n={len(v):4d} sum={sum(v)/1e3:9.1f}us mean={sum(v)/len(v)/1e3:8.1f}us")
PY
