#!/bin/bash
# quick GPU check: the -m gpu suite, then per-layer timings of the bench's VGG layers (guess)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
if [ "${TESTS:-1}" = "1" ]; then
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -rfs ${PYTEST_ARGS} > gpurun_out/pytest_quick.txt 2>&1
echo "pytest rc=$?"; tail -8 gpurun_out/pytest_quick.txt
fi
L="${LAYERS:-conv1_1 conv1_2 conv2_1 conv2_2 conv3_1 conv3_2 conv4_1 conv4_2 conv5_2}"
[ "$L" = "none" ] && L=""
for l in $L; do
  timeout 60 python scripts/layer_bench.py $l implicit_gemm --reps 20
done
