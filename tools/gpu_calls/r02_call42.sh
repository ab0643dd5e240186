#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x -k "sstep or smoke or c2_ or tstep or tgram" > gpurun_out/t42.log 2>&1 || exit 1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench42.json 2> gpurun_out/bench42.err
timeout 400 bash tools/ss_prof.sh > gpurun_out/ssprof42.log 2>&1
