#!/bin/bash
# Same-box A/B of developer knobs (libai3_dev.so, built with `python -m paper_2410_08300_b200.build --dev`):
#   scripts/ab.sh "AI3_BN=128" "AI3_BN=256" layer1 layer2 ...   (alternates A,B twice)
#   ALGO=winograd scripts/ab.sh "AI3_WINO_FUSED=1" "AI3_WINO_FUSED=0" conv1_2 conv3_2
# Knobs measured with it this round: AI3_WINO_FUSED / AI3_WINO_FUSED_KMAX / AI3_WINO_TMAJOR
# (winograd), AI3_DIRECT_ASYNC (direct), AI3_SMM_ASYNC (smm), AI3_GATHER_ASYNC
# (implicit_precomp_gemm), AI3_BN (block_n of any engine algorithm).
A="$1"; B="$2"; shift 2
ALGO=${ALGO:-guess}
REPS=${REPS:-20}
for rep in 1 2; do
  for cfg in "$A" "$B"; do
    for l in "$@"; do
      env $cfg timeout 300 python scripts/layer_bench.py $l $ALGO --reps $REPS --lib paper_2410_08300_b200/libai3_dev.so | sed "s|^|[$cfg] |"
    done
  done
done
