#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x -k "tstep or tgram or smoke or c2_" > gpurun_out/t36.log 2>&1 || exit 1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench36.json 2> gpurun_out/bench36.err
timeout 400 bash tools/tg_prof_sweep.sh 16 > gpurun_out/tgsweep36.log 2>&1
B="python tools/prof_layer.py"
timeout 300 $B > gpurun_out/plain36.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sstep_tc -s 2 -c 1 -o gpurun_out/r02_sstep36 $B > gpurun_out/ncu36a.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tgram_tc -s 2 -c 1 -o gpurun_out/r02_tgram36 $B > gpurun_out/ncu36b.log 2>&1
