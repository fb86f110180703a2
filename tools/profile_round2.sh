#!/bin/bash
# Round-2 captures of the band-formulation path (C2, one GPU): plain bench line,
# ncu launch list, one `--set full` capture per hot kernel.  Run under gpurun
# from the repo root; outputs under gpurun_out/r2prof/.
set -u
O=gpurun_out/r2prof
mkdir -p $O
CMD="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
timeout 300 $CMD > $O/plain.json 2> $O/plain.err; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_l.log 2>&1; echo "launches rc=$?"
# (band_kernel instances: K-stats then K-band of each micro-batch; skip the warm-up step's)
for spec in "band:regex:band_kernel:16:2" "gemm2:regex:gemm_grad_kernel:4:1" "adam:regex:adam_tile_kernel:4:1" \
            "lse:regex:lse_kernel:8:1" "gather:regex:gather_kernel:8:1" "pslot:regex:pslot_:16:2"; do
  IFS=: read name kind pat skip cnt <<< "$spec"
  timeout 900 ncu --set full --import-source on --clock-control none -k $kind:$pat -s $skip -c $cnt -o $O/full_$name -f $CMD > $O/ncu_$name.log 2>&1
  echo "$name rc=$?"
done
