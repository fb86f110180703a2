#!/bin/bash
# GEMM2 raster / K-chunk sweep at C2 (1 agent resident): bench time of K-GEMM2 and
# the DRAM bytes of one launch (ncu), to see whether operand re-reads cost
# power-capped clock.  Output: gpurun_out/g2_sweep.jsonl
set -u
mkdir -p gpurun_out
OUT=gpurun_out/g2_sweep.jsonl
: > $OUT
B="python bench.py --no-cpu-baseline --tier resident --agents 1 --steps 6 --warmup 3 --e2e-steps 0"
for cfg in "8 0" "1 0" "2 0" "4 0" "16 0" "1 8192" "1 4096" "8 8192"; do
  set -- $cfg
  G=$1; KC=$2
  if [ "$KC" = 0 ]; then KCE=""; else KCE="FM_G2_KCHUNK=$KC"; fi
  for rep in 1 2; do
    res=$(env FM_G2_GROUP_M=$G $KCE timeout 300 $B 2>/dev/null | tail -1)
    echo "{\"group_m\": $G, \"kchunk\": $KC, \"rep\": $rep, \"res\": $res}" >> $OUT
  done
  env FM_G2_GROUP_M=$G $KCE timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_tn_2sm -s 9 -c 2 --csv python bench.py --no-cpu-baseline --tier resident --agents 1 --steps 1 --warmup 1 --e2e-steps 0 > gpurun_out/g2_ncu_${G}_${KC}.csv 2>/dev/null
done
echo sweep-done
