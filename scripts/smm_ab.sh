# smm: asynchronous vs synchronous footprint staging (dev knob AI3_SMM_ASYNC)
for l in ${LAYERS:-conv1_2 conv3_2 conv4_2}; do
  for f in 1 0; do
    echo -n "[async=$f] "; AI3_SMM_ASYNC=$f timeout 300 python scripts/layer_bench.py $l smm --reps 3 --lib paper_2410_08300_b200/libai3_dev.so
  done
done
