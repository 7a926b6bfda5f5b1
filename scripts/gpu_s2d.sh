#!/bin/bash
# s2d lowering check: parity tests, then stem / AlexNet conv1 timing (s2d on vs off).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_s2d_gpu.py tests/test_parity_gpu.py -q -x 2>&1 | tail -8
for L in rn50_00_3x224_64_7x7s2; do
  timeout 120 python scripts/layer_bench.py $L implicit_gemm gemm --net resnet50 --batch 256 --reps 20
  AI3_S2D=0 timeout 120 python scripts/layer_bench.py $L implicit_gemm --net resnet50 --batch 256 --reps 20
done
timeout 120 python scripts/layer_bench.py conv1 implicit_gemm gemm --net alexnet --batch 128 --reps 20
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2d_launches.csv \
  python scripts/layer_bench.py rn50_00_3x224_64_7x7s2 implicit_gemm --net resnet50 --batch 256 --reps 2 > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open("gpurun_out/s2d_launches.csv")) if len(r)>10]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
for r in rows[1:]: print(r[ki][:60], r[vi])
PY
