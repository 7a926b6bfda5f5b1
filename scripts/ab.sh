#!/bin/bash
# Same-box A/B: scripts/ab.sh "ENV_A" "ENV_B" layer1 layer2 ...   (alternates A,B twice)
A="$1"; B="$2"; shift 2
for rep in 1 2; do
  for cfg in "$A" "$B"; do
    for l in "$@"; do
      env $cfg timeout 60 python scripts/layer_bench.py $l guess --reps 20 | sed "s|^|[$cfg] |"
    done
  done
done
