#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/gpu_suite12.log 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench12.json 2> gpurun_out/bench12.err
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-lut"
$B > gpurun_out/plain12.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sstep_tc -s 5 -c 1 -o gpurun_out/r02_sstep_v2 $B > gpurun_out/ncu12.log 2>&1
