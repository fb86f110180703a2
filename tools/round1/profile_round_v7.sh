#!/bin/bash
# Round-1 v7 captures (session 3 end: segmented GEMM2, 8-warp GEMM1 epilogue).
set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/v7_plain.json 2> gpurun_out/v7_plain.err; echo "plain rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v7.csv $CMD > gpurun_out/v7_ncu_l.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_tn_2sm -s 4 -c 2 -o gpurun_out/prof7_gemm -f $CMD > gpurun_out/v7_ncu_gemm.log 2>&1; echo "gemm rc=$?"
