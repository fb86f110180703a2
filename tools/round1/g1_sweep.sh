#!/bin/bash
# GEMM1 raster sweep at C2 (1 agent resident): bench time of K-GEMM1 (2 reps) and
# the DRAM bytes / duration of one launch under ncu.  Output gpurun_out/g1_sweep.jsonl
set -u
mkdir -p gpurun_out
OUT=gpurun_out/g1_sweep.jsonl
: > $OUT
B="python bench.py --no-cpu-baseline --tier resident --agents 1 --steps 6 --warmup 3 --e2e-steps 0"
for G in 16 1 2 4 8; do
  for rep in 1 2; do
    echo "{\"g1\": $G, \"rep\": $rep, \"res\": $(FM_G1_GROUP_M=$G timeout 300 $B 2>/dev/null | tail -1)}" >> $OUT
  done
  FM_G1_GROUP_M=$G timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_tn_2sm -s 8 -c 1 --csv python bench.py --no-cpu-baseline --tier resident --agents 1 --steps 1 --warmup 1 --e2e-steps 0 > gpurun_out/g1_ncu_$G.csv 2>/dev/null
done
echo sweep-done
