#!/bin/bash
# ncu evidence for profiles/ (under gpurun): (1) launch list of one bench step; (2) full capture
# of the 13 tc_gemm launches of one bench step (traffic per launch); (3) full capture of one
# execute of conv1_2 and conv3_2 for every algorithm.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
# the full captures are large: they stay in $PROF_RUN on the box; only the summaries come back
export PROF_RUN=${PROF_RUN:-/tmp/prof}
mkdir -p $PROF_RUN
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $PROF_RUN/launches.csv \
   python bench.py --quick --steps 2 --warmup 3 --no-e2e --no-cpu --no-model --no-config5 > /dev/null 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_gemm -s 39 -c 13 \
   -o $PROF_RUN/prof_step -f python bench.py --quick --steps 1 --warmup 3 --no-e2e --no-cpu --no-model --no-config5 \
   > $PROF_RUN/ncu_step.log 2>&1
echo "step capture rc=$?"
for layer in ${LAYERS:-conv1_2 conv3_2}; do
  for algo in ${ALGOS:-implicit_gemm implicit_precomp_gemm winograd gemm kn2row direct smm}; do
    timeout 600 ncu --set full --clock-control none --profile-from-start off -o $PROF_RUN/prof_${layer}_${algo} -f \
       python scripts/prof_layer.py $layer $algo > $PROF_RUN/ncu_${layer}_${algo}.log 2>&1
    echo "$layer $algo rc=$?"
  done
done
PROF_OUT=gpurun_out/profiles python scripts/summarize_r02.py ${TAG:-r02} > gpurun_out/summarize.log 2>&1
echo "summarize rc=$?"; tail -3 gpurun_out/summarize.log
cp $PROF_RUN/launches.csv gpurun_out/launches.csv 2>/dev/null
