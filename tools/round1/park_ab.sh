#!/bin/bash
# C2 N=1 (4 agents, device tier): swap-out fused into K-adam (--park fused, default)
# vs the copy-out after the update (--park copy), alternating on one box.
set -u
mkdir -p gpurun_out
OUT=gpurun_out/park_ab.jsonl
: > $OUT
B="python bench.py --no-cpu-baseline"
for rep in 1 2 3; do
  echo "{\"park\": \"fused\", \"res\": $(timeout 300 $B --park fused 2>/dev/null | tail -1)}" >> $OUT
  echo "{\"park\": \"copy\", \"res\": $(timeout 300 $B --park copy 2>/dev/null | tail -1)}" >> $OUT
done
echo "{\"park\": \"resident\", \"res\": $(timeout 300 $B --tier resident 2>/dev/null | tail -1)}" >> $OUT
echo ab-done
