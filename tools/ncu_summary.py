"""Condense ncu output into the small summaries committed under profiles/.

  python tools/ncu_summary.py launches <launches.csv> <out.json> [kernel-regex]
      per-kernel launch counts / total and mean gpu__time_duration from an
      `ncu --metrics gpu__time_duration.sum --csv` launch list, plus the
      share of the matching kernel among the launches after the first one.
  python tools/ncu_summary.py full <report.ncu-rep> <out.json> [label] [kernel-regex]
      selected counters of a `ncu --set full` capture (one launch), read
      with `ncu -i ... --page raw --csv`; `dram_bytes_per_launch` is what
      bench.py reports as roofline.traffic.
"""
from __future__ import annotations

import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict

FULL_METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__bytes_read.sum.per_second",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpc__cycles_elapsed.max",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "lts__t_bytes.sum",
    "lts__t_sector_hit_rate.pct",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block",
    "launch__grid_size",
    "launch__block_size",
    "launch__occupancy_limit_shared_mem",
    "launch__occupancy_limit_registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
]


def _num(v: str):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return v


def launches(path: str, out: str, pattern: str = "countsketch") -> None:
    text = open(path, encoding="utf-8", errors="replace").read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per = defaultdict(lambda: {"launches": 0, "total_us": 0.0})
    seq = []
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        unit = r["Metric Unit"]
        t = float(r["Metric Value"].replace(",", ""))
        t_us = t / 1000.0 if unit == "ns" else (t * 1000.0 if unit == "ms" else t)
        short = re.sub(r"\(.*", "", name)[:120]
        per[short]["launches"] += 1
        per[short]["total_us"] += t_us
        seq.append((short, t_us))
    rx = re.compile(pattern)
    hits = [t for n, t in seq if rx.search(n)]
    first = next((i for i, (n, _) in enumerate(seq) if rx.search(n)), None)
    after = seq[first:] if first is not None else []
    summary = {
        "source": path,
        "kernel_pattern": pattern,
        "kernel_launches": len(hits),
        "kernel_mean_us": round(sum(hits) / len(hits), 3) if hits else None,
        "kernel_min_us": round(min(hits), 3) if hits else None,
        "kernel_share_from_first_launch": (round(sum(hits) / sum(t for _, t in after), 4)
                                           if after else None),
        "note": "ncu per-launch times are serialised and cold-cache (--clock-control none); "
                "compare shares, not absolutes, with bench.py's CUDA-event timings",
        "kernels": {k: {"launches": v["launches"], "total_us": round(v["total_us"], 2),
                        "mean_us": round(v["total_us"] / v["launches"], 3)}
                    for k, v in sorted(per.items(), key=lambda kv: -kv[1]["total_us"])},
    }
    json.dump(summary, open(out, "w"), indent=1)
    print(json.dumps({k: summary[k] for k in list(summary)[:6]}))


def full(rep: str, out: str, label: str = "", kernel: str = "") -> None:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    # the first launch whose kernel name matches (all launches when no regex)
    ki = hdr.index("Kernel Name")
    vals = next(r for r in rows[2:] if not kernel or re.search(kernel, r[ki]))
    got = {}
    for h, u, v in zip(hdr, units, vals):
        if h in FULL_METRICS or h in ("Kernel Name", "Block Size", "Grid Size"):
            got[h] = {"value": _num(v), "unit": u} if u else _num(v)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}

    def to_bytes(key):
        e = got.get(key)
        return e["value"] * scale.get(e["unit"], 1) if isinstance(e, dict) else None

    rd, wr = to_bytes("dram__bytes_read.sum"), to_bytes("dram__bytes_write.sum")
    summary = {"label": label, "report": rep,
               "dram_bytes_per_launch": (rd + wr) if rd is not None and wr is not None else None,
               "metrics": got}
    json.dump(summary, open(out, "w"), indent=1)
    print(out, "dram_bytes_per_launch", summary["dram_bytes_per_launch"])


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(*sys.argv[2:])
    elif sys.argv[1] == "full":
        full(*sys.argv[2:])
    else:
        raise SystemExit(__doc__)
