#!/bin/bash
cd "$(dirname "$0")/.."
python - <<'PY' 2>&1 | grep -v "^$"
import os, sys, subprocess
sys.path.insert(0, ".")
from synth import workload
for net, b in (("resnet50", 256), ("alexnet", 128), ("vgg16", 64)):
    for l in workload(net, b):
        r = subprocess.run([sys.executable, "scripts/layer_bench.py", l.name, "guess", "--net", net, "--batch", str(b), "--reps", "10"],
                           capture_output=True, text=True, env=dict(os.environ, AI3_TC_VERBOSE="1"))
        cfg = sorted(set(x for x in r.stderr.splitlines() if "[ai3 tc]" in x))
        print(r.stdout.strip(), "|", cfg[0].replace("[ai3 tc] ", "") if cfg else r.stderr[-200:])
PY
