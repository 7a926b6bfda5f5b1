#!/bin/bash
# Same-box A/B of two builds of libai3.so on a few VGG layers: scripts/ab_lib.sh OLD.so
OLD="$1"; shift
for rep in 1 2; do
  for lib in "$OLD" paper_2410_08300_b200/libai3.so; do
    for l in ${LAYERS:-conv1_2 conv3_2 conv5_2}; do
      timeout 60 python scripts/layer_bench.py $l implicit_gemm --reps 20 --lib $lib | sed "s|^|[$(basename $lib)] |"
    done
  done
done
