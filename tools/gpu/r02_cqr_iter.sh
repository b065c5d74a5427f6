timeout 300 python -m pytest tests/test_gpu_cholqr.py -q 2>&1 | grep -E "passed|failed|Error|assert" | head -20
timeout 200 python tools/time_cholqr.py 2048x256 800x200 2048x511 2>&1 | tail -3
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv -k regex:cqr \
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
export SKL_NVCC_DEFINES=-DSKL_CQR_PROBE
python -c "from paper_2409_14309_b200 import _build; _build.build(force=True)" 2>&1 | tail -2
timeout 120 python tools/probe_cholqr.py 2048x256 2>&1 | head -11 | cut -c1-200
