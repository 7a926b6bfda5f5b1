#!/bin/bash
cd "$(dirname "$0")/.."
for l in conv1_1 conv1_2; do timeout 60 python scripts/trace_layer.py $l; done
