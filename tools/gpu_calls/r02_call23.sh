#!/bin/bash
# tgram_tc: per-role cycle accounting (KPROF build) and one ncu --set full capture with source
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
bash tools/tg_prof.sh > gpurun_out/tgprof23.log 2>&1
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-lut"
$B > gpurun_out/plain23.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:tgram_tc -s 3 -c 1 \
    -o gpurun_out/r02_tgram $B > gpurun_out/ncu23.log 2>&1
