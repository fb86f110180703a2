#!/bin/bash
# GEMM1 raster in the segmented-GEMM2 layout (C2, 1 agent resident): bench 2 reps +
# one ncu launch (DRAM bytes, duration, clock) per group size.  gpurun_out/g1seg_*.
set -u
mkdir -p gpurun_out
OUT=gpurun_out/g1seg_sweep.jsonl
: > $OUT
B="python bench.py --no-cpu-baseline --tier resident --agents 1 --steps 6 --warmup 3 --e2e-steps 0"
for G in 16 8 32 12; do
  for rep in 1 2; do
    echo "{\"g1\": $G, \"rep\": $rep, \"res\": $(FM_G1_GROUP_M=$G timeout 300 $B 2>/dev/null | tail -1)}" >> $OUT
  done
  FM_G1_GROUP_M=$G timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:LogitsEpi -s 4 -c 1 --csv python bench.py --no-cpu-baseline --tier resident --agents 1 --steps 1 --warmup 1 --e2e-steps 0 > gpurun_out/g1seg_ncu_$G.csv 2>/dev/null
done
echo sweep-done
