#!/bin/bash
# GEMM raster sweep (run under gpurun on one B200): m-tiles per raster group for
# K-GEMM1 / K-GEMM2 (FM_G1_GROUP_M / FM_G2_GROUP_M), one resident C2 agent, then
# GEMM2's long-K case (C5, K = 65,536 rows at N=1).  One JSON line per run.
set -u
mkdir -p gpurun_out
OUT=gpurun_out/raster_sweep.jsonl
: > $OUT
B="python bench.py --agents 1 --tier resident --steps 6 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
for g in 2 4 8 16 32 125; do
  echo "{\"g2\": $g, \"res\": $(FM_G2_GROUP_M=$g timeout 300 $B 2>/dev/null | tail -1)}" >> $OUT
done
for g in 4 8 32 64; do
  echo "{\"g1\": $g, \"res\": $(FM_G1_GROUP_M=$g timeout 300 $B 2>/dev/null | tail -1)}" >> $OUT
done
C5="python bench.py --config C5 --agents 1 --tier resident --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
for g in 4 8 16; do
  echo "{\"c5_g2\": $g, \"res\": $(FM_G2_GROUP_M=$g timeout 600 $C5 2>/dev/null | tail -1)}" >> $OUT
done
