#!/bin/bash
# (experiment record: the FM_G1_POL / FM_G2_POL knobs it sets were removed after the sweep)
# L2 eviction-priority x raster sweep at C2 (1 agent resident): one GEMM1 + one
# GEMM2 launch under ncu (DRAM bytes, duration, SM clock) per configuration.
set -u
mkdir -p gpurun_out
C="python bench.py --no-cpu-baseline --tier resident --agents 1 --steps 1 --warmup 1 --e2e-steps 0"
for cfg in "16 00 1 00" "16 01 1 10" "32 01 1 10" "64 01 1 10" "8 01 8 10" "32 00 2 10"; do
  set -- $cfg
  tag="g1_$1_p$2_g2_$3_p$4"
  FM_G1_GROUP_M=$1 FM_G1_POL=$2 FM_G2_GROUP_M=$3 FM_G2_POL=$4 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_tn_2sm -s 8 -c 2 --csv $C > gpurun_out/pol_$tag.csv 2>/dev/null
  echo "$tag rc=$?"
done
echo sweep-done
