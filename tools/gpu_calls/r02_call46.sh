#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x -k "sstep or smoke or c2_ or tstep or tgram" > gpurun_out/t46.log 2>&1 || exit 1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench46.json 2> gpurun_out/bench46.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench46b.json 2> gpurun_out/bench46b.err
timeout 400 bash tools/tg_prof_sweep.sh 16 > gpurun_out/tgsweep46.log 2>&1
