#!/bin/bash
# DP-gang sweep: one agent on a gang of N GPUs (fused GEMM2 reduce-scatter +
# sharded Adam), C3 and C5, N = 1, 2, 4 (as many GPUs as the box has).
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
for c in C3 C5; do
  for n in 1 2 4; do
    [ $n -gt $NG ] && continue
    out=gpurun_out/dp_${c}_$n.json
    if [ $n -eq 1 ]; then
      timeout 600 python bench.py --config $c --agents 1 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $out 2> ${out%.json}.err
    else
      timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n \
        bench.py --gpus $n --config $c --agents 1 --steps 3 --warmup 3 --e2e-steps 0 > $out 2> ${out%.json}.err
    fi
    echo "$c n=$n rc=$? $(python -c "import json;d=json.loads(open('$out').read().strip().splitlines()[-1]);print(round(d['value']), round(d['ms_per_step'],1))" 2>/dev/null)"
  done
done
