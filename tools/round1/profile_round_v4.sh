#!/bin/bash
# Round-1 v4 captures (under gpurun, one B200): plain bench, launch list, K-lse,
# the on-device table kernels, and a GEMM2 raster A/B at the long-K C5 shape.
set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err; echo "plain rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v4.csv $CMD > gpurun_out/ncu_l.log 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lse_kernel -s 4 -c 1 -o gpurun_out/prof4_lse -f $CMD > gpurun_out/ncu_lse.log 2>&1; echo "lse rc=$?"
timeout 120 python tools/dtable_probe.py > gpurun_out/dtable_plain.log 2>&1; echo "dtable plain rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_dtable.csv python tools/dtable_probe.py > gpurun_out/ncu_dt_l.log 2>&1; echo "dtable launches rc=$?"
for k in poll_small_kernel chunk_candidates_kernel rank_kernel release_kernel; do
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:$k -s 2 -c 1 -o gpurun_out/prof4_$k -f python tools/dtable_probe.py > gpurun_out/ncu_$k.log 2>&1; echo "$k rc=$?"
done
C5="python bench.py --config C5 --agents 1 --tier resident --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
: > gpurun_out/c5_raster_ab.jsonl
for rep in 1 2; do for g in 8 16 32; do
  echo "{\"g2\": $g, \"res\": $(FM_G2_GROUP_M=$g timeout 600 $C5 2>/dev/null | tail -1)}" >> gpurun_out/c5_raster_ab.jsonl
done; done
