#!/bin/bash
# Round profile capture (run under gpurun on one B200): plain bench first, then
# the ncu launch list of the same command, then one full capture per hot kernel.
set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
ONLY=${1:-all}
if [ "$ONLY" = all ]; then
timeout 300 $CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err; echo "plain rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v3.csv $CMD > gpurun_out/ncu_l.log 2>&1; echo "launches rc=$?"
for k in adam_kernel lse_kernel gather_kernel; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 4 -c 1 -o gpurun_out/prof3_$k -f $CMD > gpurun_out/ncu_$k.log 2>&1; echo "$k rc=$?"
done
fi
# GEMM1 + GEMM2 of the third micro-batch (launch names carry no template args)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_tn_2sm -s 4 -c 2 -o gpurun_out/prof3_gemm -f $CMD > gpurun_out/ncu_gemm.log 2>&1; echo "gemm rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:colmax -s 1 -c 1 -o gpurun_out/prof3_colmax -f $CMD > gpurun_out/ncu_colmax.log 2>&1; echo "colmax rc=$?"
