#!/bin/bash
cd "$(dirname "$0")/.."
for L in rn50_04_256x56_64_1x1s1 rn50_09_512x28_128_1x1s1 rn50_00_3x224_64_7x7s2; do timeout 60 python scripts/trace_layer.py $L resnet50 2>&1 | tail -12; done
timeout 60 python scripts/trace_layer.py conv1_1 vgg16 2>&1 | tail -12
