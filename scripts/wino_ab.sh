# Winograd A/B (dev knobs: AI3_WINO_FUSED, AI3_WINO_FUSED_KMAX, AI3_WINO_TMAJOR) per layer
mkdir -p gpurun_out
for l in ${LAYERS:-conv2_2 conv3_2 conv4_2}; do
  for cfg in ${CFGS:-"AI3_WINO_TMAJOR=0" "AI3_WINO_TMAJOR=1"}; do
    echo -n "[$cfg] "; env $cfg timeout 120 python scripts/layer_bench.py $l winograd --reps 10 --lib paper_2410_08300_b200/libai3_dev.so
  done
done
