#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over scripts/sanitize_cases.py
# (under gpurun); summaries in gpurun_out/sanitize_<tool>.txt.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  timeout ${T_SAN:-1500} compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
      python scripts/sanitize_cases.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitize_$tool.txt
done
