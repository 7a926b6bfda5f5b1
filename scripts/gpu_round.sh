#!/bin/bash
# One GPU session: tests, bench, ncu launch list, one full ncu capture of the top kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2410_08300_b200.build > /dev/null
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/bench.err
cat gpurun_out/bench.json
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-e2e --no-compare --no-cpu --no-model --no-configs > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 16 -c 2 -o gpurun_out/prof_tc -f \
   python bench.py --steps 1 --warmup 3 --no-e2e --no-compare --no-cpu --no-model --no-configs > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -3 gpurun_out/ncu_full.log
fi
