#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "tstep or tgram or smoke or c2_ or free_running" > gpurun_out/t26.log 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench26.json 2> gpurun_out/bench26.err
bash tools/tg_prof_sweep.sh 16 17 18 20 > gpurun_out/tgsweep26.log 2>&1
