# fused vs unfused Winograd A/B (dev knobs: AI3_WINO_FUSED, AI3_WINO_FUSED_KMAX) per layer
mkdir -p gpurun_out
for l in ${LAYERS:-conv1_1 conv1_2 conv2_2 conv3_2 conv4_2}; do
  for cfg in "AI3_WINO_FUSED=1 AI3_WINO_FUSED_KMAX=512" "AI3_WINO_FUSED=0"; do
    echo -n "[$cfg] "; env $cfg timeout 120 python scripts/layer_bench.py $l winograd --reps 10 --lib paper_2410_08300_b200/libai3_dev.so
  done
done
