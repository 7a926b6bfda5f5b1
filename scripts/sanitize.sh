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
# racecheck with every engine launch on single-CTA tiles (dev build, AI3_TC_CG=1): separates
# hazards of the CTA-pair TMEM allocation (tcgen05.alloc.cta_group::2) from the rest
if [ "${CG1:-1}" = "1" ]; then
  AI3_TC_CG=1 timeout ${T_SAN:-1500} compute-sanitizer --tool racecheck --target-processes all --print-limit 50 \
      python scripts/sanitize_cases.py --dev > gpurun_out/sanitize_racecheck_cg1.txt 2>&1
  echo "racecheck (cg1) rc=$?"; tail -4 gpurun_out/sanitize_racecheck_cg1.txt
fi
