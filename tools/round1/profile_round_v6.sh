#!/bin/bash
# Round-1 v6 captures (session 3, segmented GEMM2 default; under gpurun, one B200):
# plain bench, the ncu launch list of the same command, full captures of the hot kernels.
set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/v6_plain.json 2> gpurun_out/v6_plain.err; echo "plain rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v6.csv $CMD > gpurun_out/v6_ncu_l.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_tn_2sm -s 4 -c 2 -o gpurun_out/prof6_gemm -f $CMD > gpurun_out/v6_ncu_gemm.log 2>&1; echo "gemm rc=$?"
for k in adam_kernel kslot_place_kernel kslot_count_kernel gather_kernel; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 2 -c 1 -o gpurun_out/prof6_$k -f $CMD > gpurun_out/v6_ncu_$k.log 2>&1; echo "$k rc=$?"
done
