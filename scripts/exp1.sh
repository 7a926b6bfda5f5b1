#!/bin/bash
# experiment batch: HBM write ceiling by store method; conv5 N-tile A/B; conv1_1 / conv1_2 timing
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
./scripts/micro/hbm_write > gpurun_out/hbm_write.txt 2>&1; cat gpurun_out/hbm_write.txt
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
DEV=paper_2410_08300_b200/libai3_dev.so
for rep in 1 2; do
for cfg in "AI3_N2=1" "AI3_N2=0 AI3_BN=192" "AI3_N2=0 AI3_BN=128" "AI3_N2=0 AI3_BN=256" "AI3_N2=0 AI3_BN=96"; do
  env $cfg timeout 60 python scripts/layer_bench.py conv5_2 implicit_gemm --reps 20 --lib $DEV | sed "s|^|[$cfg] |"
done
done
for l in conv1_1 conv1_2 conv2_1 conv3_1; do timeout 60 python scripts/layer_bench.py $l implicit_gemm --reps 20; done
