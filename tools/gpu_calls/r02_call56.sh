#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
L="python tools/prof_layer.py"
timeout 300 $L > gpurun_out/plain56.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:trhs -s 2 -c 1 -o gpurun_out/r02_trhs $L > gpurun_out/ncu56.log 2>&1
