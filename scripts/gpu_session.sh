#!/bin/bash
# One GPU session (under gpurun): build, the -m gpu suite, the default bench line, and the
# ncu launch list of one bench step.  Outputs land in gpurun_out/.
#   TESTS=0 / BENCH=0 / NCU=0 skip a part; PYTEST_ARGS adds pytest arguments.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo "build failed"; tail -20 gpurun_out/build.log; exit 1; }
if [ "${TESTS:-1}" = "1" ]; then
  timeout ${T_TESTS:-1500} python -m pytest tests -m gpu -q ${XFLAG} --timeout 600 --timeout-method thread -rfs --durations=30 \
      ${PYTEST_ARGS} > gpurun_out/pytest_gpu_full.txt 2>&1
  echo "pytest rc=$?"
  tail -45 gpurun_out/pytest_gpu_full.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.txt
fi
if [ "${BENCH:-1}" = "1" ]; then
  nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks.csv &
  SMI=$!
  timeout ${T_BENCH:-900} python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
  kill $SMI 2>/dev/null
  tail -5 gpurun_out/bench.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print({k: d.get(k) for k in ('value','ms_per_step','roofline','clocks')})
print('per_algorithm', d.get('per_algorithm')); print('e2e', d.get('e2e'))
for k in ('peaks','fp32_stack','config1_latency_us','dispatch_overhead','vgg16_model','config5','selector_quality'): print(k, d.get(k))
" 2>&1 | cut -c1-3000
fi
if [ "${NCU:-1}" = "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
     python bench.py --steps 2 --warmup 3 --quick --no-e2e --no-cpu --no-model --no-config5 > gpurun_out/ncu_bench_stdout.txt 2>&1
  echo "ncu launch list rc=$?"
fi
