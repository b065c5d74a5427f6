#!/bin/bash
# Config-1 CountSketch (20000x200, d=800) ring-geometry sweep: plan chunk x
# ring stages through the A/B knobs SKL_OWNED_CHUNK / SKL_OWNED_STAGES.
out=${1:-gpurun_out/sweep_cfg1.jsonl}
: > "$out"
for ch in 0 256 512 1024 2048; do
  for st in 0 2 3 4 6; do
    r=$(SKL_OWNED_CHUNK=$ch SKL_OWNED_STAGES=$st timeout 120 python tools/bench_configs.py --configs 1 --reps 30 2>/dev/null | tail -1)
    echo "{\"chunk\": $ch, \"stages\": $st, \"r\": $r}" >> "$out"
  done
done
