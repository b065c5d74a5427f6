"""Top SASS instructions by warp-stall samples from an ncu report (source
page), with the stall-reason columns that dominate them.
  python tools/ncu_hot.py <report.ncu-rep> <kernel-regex> [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
end = next((i for i, r in enumerate(rows[1:], 1) if r and r[0] == "Kernel Name"), len(rows))
rows = [r for r in rows[:end] if len(r) > 2]
si = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h and i != si]
tot = sum(float(r[si] or 0) for r in rows[1:] if len(r) > si)
print(f"total samples {tot:.0f}")
best = sorted(rows[1:], key=lambda r: -float(r[si] or 0))[:top]
for r in best:
    print(f"{float(r[si]):7.0f} {100 * float(r[si]) / tot:5.1f}%  {r[0][-5:]}  {r[1].strip()[:70]}")
