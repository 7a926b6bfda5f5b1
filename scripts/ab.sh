#!/bin/bash
# Same-box A/B of developer knobs (libai3_dev.so, built with `python -m paper_2410_08300_b200.build --dev`):
#   scripts/ab.sh "AI3_BN=128" "AI3_BN=256" layer1 layer2 ...   (alternates A,B twice)
A="$1"; B="$2"; shift 2
for rep in 1 2; do
  for cfg in "$A" "$B"; do
    for l in "$@"; do
      env $cfg timeout 60 python scripts/layer_bench.py $l guess --reps 20 --lib paper_2410_08300_b200/libai3_dev.so | sed "s|^|[$cfg] |"
    done
  done
done
