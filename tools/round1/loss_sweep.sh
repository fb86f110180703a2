#!/bin/bash
# BASELINE config 5: "vocab 128k, seq 4096 fused loss-kernel stress sweep at 1/2/4/8 B200".
# One agent, V=128,000, D=8,192; a DP gang of N GPUs trains M/N rows of each
# 16 x 4,096-token micro-batch per GPU, so the per-GPU loss kernels of N=1/2/4/8
# are measured at 65,536 / 32,768 / 16,384 / 8,192 rows (--resp-len 4096/N).
# Both loss formulations: the default fold (K-lse + gradient folded into GEMM2's
# operands) and FM_LOSS_FOLD=0 (the standalone fused log-softmax-gradient pass
# K-loss: TMA-staged p~ tiles in, G^T tiles out).
set -u
mkdir -p gpurun_out
OUT=gpurun_out/loss_sweep.jsonl
: > $OUT
for fold in 1 0; do for L in 4096 2048 1024 512; do
  r=$(FM_LOSS_FOLD=$fold timeout 900 python bench.py --config C5 --agents 1 --tier resident --resp-len $L \
      --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | tail -1)
  echo "{\"fold\": $fold, \"resp_len\": $L, \"res\": ${r:-null}}" >> $OUT
done; done
